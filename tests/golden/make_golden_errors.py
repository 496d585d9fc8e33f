"""Record the reference's outcome (exception class or "ok") for a list of
bad and borderline calls, so the device package can be checked for the same
error behaviour (tests/test_gpu_errors.py).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_errors.py

Cases are plain data interpreted by `run_case` below; the test replays them
with the same interpreter against paper_2211_15299_b200.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

J8 = [23, 187, 190, 247, 386, 731, 990, 994]  # reference tests/test_hidft.py:111-118 (pivots 0, 2, 5)
J5 = [3, 17, 25, 27, 35]                        # tests/test_congruence.py:140-146 (pivots 1, 3, 5)

CASES = [
    # SupportSet.make (congruence.py:52-57)
    {"op": "support", "N": 48, "J": [1, 2]},
    {"op": "support", "N": 64, "J": [5, 3]},
    {"op": "support", "N": 64, "J": [3, 3]},
    {"op": "support", "N": 64, "J": [3, 64]},
    {"op": "support", "N": 64, "J": [-1, 3]},
    {"op": "support", "N": 64, "J": []},
    {"op": "support", "N": 1, "J": [0]},
    {"op": "support", "N": 64, "J": [0]},
    # pivoted_pattern (sampling.py:62-71)
    {"op": "pattern", "r": [2, 0], "M": 10},
    {"op": "pattern", "r": [0, 10], "M": 10},
    {"op": "pattern", "r": [-1], "M": 10},
    {"op": "pattern", "r": [1, 1], "M": 10},
    {"op": "pattern", "r": [], "M": 10},
    # hidft (hidft.py:135-185)
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 0, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 0, "shift": 0, "n": 512},
    {"op": "hidft", "N": 1024, "J": J8, "r": [5, 2, 0], "height": 0, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 10], "height": 0, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [2, 5], "height": 0, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 4, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": -1, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 3, "shift": 0, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 0, "shift": -7, "n": 1024},
    {"op": "hidft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 0, "shift": 5000, "n": 1024},
    {"op": "hidft", "N": 64, "J": J5, "r": [3], "height": 0, "shift": 0, "n": 64},
    {"op": "hidft", "N": 64, "J": J5, "r": [1, 3], "height": 0, "shift": 0, "n": 64},
    {"op": "hidft", "N": 64, "J": J5, "r": [0, 1, 3], "height": 0, "shift": 0, "n": 64},
    {"op": "hidft_callable", "N": 1024, "J": J8, "r": [0, 2, 5], "ret": "short"},
    {"op": "hidft_callable", "N": 1024, "J": J8, "r": [0, 2, 5], "ret": "ok"},
    # hidft_to_dft (hidft.py:188-207)
    {"op": "to_dft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 0},
    {"op": "to_dft", "N": 1024, "J": J8, "r": [0, 2, 5], "height": 1},
    {"op": "to_dft", "N": 64, "J": J5, "r": [1, 3], "height": 0},
    {"op": "to_dft", "N": 64, "J": J5, "r": [1, 3, 5], "height": 0},
    # select_pivots / sas_transform (sas.py:89-129, 313-409)
    {"op": "select", "N": 1024, "J": J8, "policy": "bogus", "meta": None},
    {"op": "select", "N": 1024, "J": J8, "policy": "balanced", "meta": None},
    {"op": "select", "N": 1024, "J": J8, "policy": "random_subset", "meta": None},
    {"op": "select", "N": 1024, "J": J8, "policy": "uoe", "meta": None},
    {"op": "select", "N": 1024, "J": J8, "policy": "auto", "meta": None},
    {"op": "select", "N": 1024, "J": J8, "policy": "balanced", "meta": {"pivots": [0, 2, 5]}},
    {"op": "sas", "N": 1024, "J": J8, "r": [2, 0], "policy": "auto", "meta": None},
    {"op": "sas", "N": 1024, "J": J8, "r": [0, 2, 5], "policy": "auto", "meta": None},
    {"op": "sas", "N": 1024, "J": J8, "r": None, "policy": "bogus", "meta": None},
    {"op": "sas", "N": 64, "J": J5, "r": [3], "policy": "auto", "meta": None},
    {"op": "sas", "N": 64, "J": J5, "r": [1], "policy": "auto", "meta": None},
]


def run_case(S, c):
    """Evaluate one case against package S; returns "ok" or the exception class name."""
    try:
        if c["op"] == "support":
            S.SupportSet.make(c["N"], c["J"])
        elif c["op"] == "pattern":
            S.pivoted_pattern(tuple(c["r"]), c["M"])
        elif c["op"] in ("hidft", "hidft_callable", "to_dft"):
            J = S.SupportSet.make(c["N"], c["J"])
            if c["op"] == "hidft_callable":
                n = 3 if c["ret"] == "short" else None
                src = (lambda loc, n=n: np.zeros(n if n else len(loc), complex))
                S.hidft(src, J, tuple(c["r"]))
            elif c["op"] == "hidft":
                S.hidft(np.zeros(c["n"], complex), J, tuple(c["r"]), height=c["height"], shift=c["shift"])
            else:
                S.hidft_to_dft(S.hidft(np.zeros(c["N"], complex), J, tuple(c["r"]), height=c["height"]))
        elif c["op"] == "select":
            S.select_pivots(S.SupportSet.make(c["N"], c["J"]), c["policy"], c["meta"])
        elif c["op"] == "sas":
            J = S.SupportSet.make(c["N"], c["J"])
            r = None if c["r"] is None else tuple(c["r"])
            S.sas_transform(np.zeros(c["N"], complex), J, r=r, policy=c["policy"], family_meta=c["meta"])
        else:
            raise AssertionError(c["op"])
        return "ok"
    except Exception as e:  # noqa: BLE001 - the class name is the recorded outcome
        return type(e).__name__


def main() -> None:
    sys.path.insert(0, REF)
    import structfft as R
    out = []
    for c in CASES:
        d = dict(c)
        d["expect"] = run_case(R, c)
        out.append(d)
    with open(os.path.join(HERE, "error_cases.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"{len(out)} cases written; outcomes:", sorted({d['expect'] for d in out}))


if __name__ == "__main__":
    main()
