"""Digests of the UNMODIFIED reference's plan tables at the BASELINE config sizes.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_plan_digests.py

For configs 1, 2, 3, 5 (shared supports) and the first two config-4 supports
it calls the reference's own `_build_plan` (hidft.py:69-95) and `hidft`
(hidft.py:135-185; a zero signal: only the index outputs are used) and writes
`plan_digests.json`: sha256 of element_slots, slot_residues, slot_real,
node_residues and the slot-order offsets (hidft.py:155-158) as little-endian
int64 / uint8, plus 512 sampled twiddles (complex128, exact repr).  The
tables themselves are up to 2^16 entries each; the digests pin the oracle
restatement (tests/test_oracle_golden.py) and the device plan
(tests/test_gpu_parity.py) to the reference at full size.  Nothing at test
time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray, dt: str) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dt)).tobytes()).hexdigest()


def twiddle_sample_index(n: int) -> np.ndarray:
    """512 positions of the concatenated stage-major twiddle table (all of a short one)."""
    if n <= 512:
        return np.arange(n, dtype=np.int64)
    return np.unique(np.concatenate([np.arange(64), (np.arange(448) * 2654435761 % n)])).astype(np.int64)


def main() -> None:
    sys.path.insert(0, REF)
    import structfft as R
    from structfft.families import rng_from_seed
    from structfft.hidft import _build_plan

    def homog(c, P_hi, p, M):
        piv = sorted(int(x) for x in rng_from_seed(c, 7).choice(P_hi, size=p, replace=False))
        return R.gen_homogeneous(piv, M, c)

    cases = {"cfg1": (homog(1, 16, 8, 16), 16), "cfg2": (homog(2, 16, 10, 20), 20), "cfg5": (homog(5, 26, 16, 26), 26)}
    H = homog(3, 22, 14, 22)
    pick = np.sort(rng_from_seed(3, 8).choice(1 << 14, size=1 << 12, replace=False))
    cases["cfg3"] = (R.SupportSet.make(1 << 22, H.as_array()[pick].tolist()), 22)
    for b in range(2):
        piv = sorted(int(x) for x in rng_from_seed(4, 9, b).choice(16, size=10, replace=False))
        seed_b = int(rng_from_seed(4, 10, b).integers(0, 2 ** 62))
        cases[f"cfg4_b{b}"] = (R.gen_homogeneous(piv, 20, seed_b), 20)

    out = {}
    for name, (J, M) in cases.items():
        r = R.pivots(J)
        plan = _build_plan(J, r)
        res = R.hidft(lambda loc: np.zeros(len(loc), np.complex128), J, r)
        off = np.zeros(1 << len(r), dtype=np.int64)
        for i, rk in enumerate(r):  # hidft.py:155-158
            off += ((np.arange(1 << len(r)) >> i) & 1) << (M - 1 - rk)
        tw = np.concatenate(plan.twiddles) if plan.twiddles else np.zeros(0, np.complex128)
        idx = twiddle_sample_index(tw.size)
        out[name] = {
            "M": M, "k": len(J), "pivots": [int(x) for x in r], "level": int(res.level),
            "sha256": {
                "J": digest(J.as_array(), "<i8"),
                "element_slots": digest(plan.element_slots, "<i8"),
                "slot_residues": digest(res.slot_residues, "<i8"),
                "slot_real": digest(np.asarray(res.slot_real, bool), "u1"),
                "node_residues": digest(res.node_residues, "<i8"),
                "offsets": digest(off, "<i8"),
            },
            "twiddle_count": int(tw.size),
            "twiddle_sample": [[float(z.real).hex(), float(z.imag).hex()] for z in tw[idx]],
        }
        print(name, "k", len(J), "s", len(r), "twiddles", tw.size)
    with open(os.path.join(HERE, "plan_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
