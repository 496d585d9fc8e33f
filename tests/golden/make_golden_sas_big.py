"""Golden shift-and-sample cases with node weight mu* > 64 from the UNMODIFIED
reference (the device decoder's CTA-per-node path).

    python tests/golden/make_golden_sas_big.py      (needs /root/reference)

Cases: a single node of weight 100 (pivot vector (), i.e. the k x k
Vandermonde of the submatrix method) and random subsets whose "uoe" / explicit
pivot prefixes leave nodes of weight 65-160, band-limited sources.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import structfft as R
    rng = np.random.default_rng(9001)
    cases = []
    J = R.SupportSet.make(1 << 10, sorted(rng.choice(1 << 10, size=100, replace=False).tolist()))
    cases.append((J, ()))
    for M, k, t in ((12, 300, 2), (13, 600, 3), (11, 140, 1)):
        J = R.SupportSet.make(1 << M, sorted(rng.choice(1 << M, size=k, replace=False).tolist()))
        p = R.pivots(J)
        cases.append((J, tuple(p[:t])))
    out = {}
    for i, (J, r) in enumerate(cases):
        mag = 0.5 + rng.random(len(J))
        c = mag * np.exp(1j * rng.random(len(J)) * 2 * np.pi)
        sig = R.BandlimitedSignal(J, c)
        res = R.sas_transform(sig, J, r=r, policy="balanced", family_meta={"pivots": r})
        rep = res.report
        pre = f"b{i}_"
        out[pre + "N"] = np.asarray([J.N])
        out[pre + "J"] = J.as_array()
        out[pre + "c"] = c
        out[pre + "r"] = np.asarray(r, np.int64)
        out[pre + "plan"] = np.asarray([res.plan.decode_level, res.plan.mu_star], np.int64)
        out[pre + "weights"] = np.asarray(res.plan.node_weights, np.int64)
        out[pre + "coeffs"] = res.coeffs
        out[pre + "report"] = np.asarray([rep.escalated_nodes, rep.dense_fallbacks], np.int64)
        print(i, "k", len(J), "r", r, "mu*", res.plan.mu_star, "escalated", rep.escalated_nodes,
              "fallbacks", rep.dense_fallbacks, "err vs planted", float(np.max(np.abs(res.coeffs - c))))
    out["n_cases"] = np.asarray([len(cases)])
    np.savez_compressed(os.path.join(HERE, "golden_sas_big.npz"), **out)


if __name__ == "__main__":
    main()
