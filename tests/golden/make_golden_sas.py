"""Golden vectors for shift-and-sample (mu* > 1) from the UNMODIFIED reference.

    python tests/golden/make_golden_sas.py      (needs /root/reference)

Cases follow the reference's tests/test_sas.py shapes: the worked 2x2 example,
the union-of-elementary fixtures with policy "uoe", random small supports
under the "auto" policy, and random subsets of homogeneous sets under
"auto" and "random_subset" (where double-double escalation happens), with
band-limited (planted) and dense sources.
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
    from structfft.bench import FIXTURES

    rng = np.random.default_rng(4243)
    cases = []  # (J, policy, meta, dense)
    cases.append((R.SupportSet.make(1024, [0, 1, 6, 7, 512]), "auto", None, False))
    cases.append((R.SupportSet.make(*FIXTURES["uoe_union"]), "uoe", None, False))
    cases.append((R.SupportSet.make(*FIXTURES["uoe_adversarial"]), "uoe", None, False))
    for _ in range(16):
        M = int(rng.integers(4, 11))
        N = 1 << M
        k = int(rng.integers(2, 17))
        cases.append((R.SupportSet.make(N, rng.choice(N, size=k, replace=False).tolist()), "auto", None,
                      bool(rng.integers(0, 2))))
    for _ in range(16):
        M = int(rng.integers(3, 11))
        N = 1 << M
        k = int(rng.integers(1, min(N, 40) + 1))
        cases.append((R.SupportSet.make(N, rng.choice(N, size=k, replace=False).tolist()), "auto", None,
                      bool(rng.integers(0, 2))))
    for seed, (M, p, kk) in enumerate([(12, 7, 48), (14, 8, 96), (16, 9, 160), (16, 10, 300)]):
        base = tuple(sorted(rng.choice(M, size=p, replace=False).tolist()))
        H = R.gen_homogeneous(base, M, 100 + seed)
        idx = np.sort(rng.choice(len(H), size=kk, replace=False))
        J = R.SupportSet.make(H.N, H.as_array()[idx].tolist())
        for pol in ("auto", "random_subset"):
            cases.append((J, pol, {"base_pivots": base}, pol == "auto"))
    out: dict[str, np.ndarray] = {}
    kept = 0
    for J, pol, meta, dense in cases:
        mag = 0.5 + rng.random(len(J))
        c = mag * np.exp(1j * rng.random(len(J)) * 2 * np.pi)
        sig = R.BandlimitedSignal(J, c)
        src = sig.synthesize() if dense and J.N <= 1 << 16 else sig
        ctr = R.OpCounter()
        res = R.sas_transform(src, J, policy=pol, family_meta=meta, counter=ctr)
        if res.plan.mu_star > 64:
            continue
        p = f"s{kept}_"
        kept += 1
        rep = res.report
        out[p + "N"] = np.asarray([J.N])
        out[p + "J"] = J.as_array()
        out[p + "c"] = c
        out[p + "dense"] = np.asarray([int(src is not sig)])
        out[p + "policy"] = np.frombuffer(pol.encode().ljust(16), np.uint8)
        out[p + "base"] = np.asarray((meta or {}).get("base_pivots", ()), np.int64)
        out[p + "pivots"] = np.asarray(res.plan.pivots, np.int64)
        out[p + "plan"] = np.asarray([res.plan.decode_level, res.plan.mu_star], np.int64)
        out[p + "weights"] = np.asarray(res.plan.node_weights, np.int64)
        out[p + "coeffs"] = res.coeffs
        out[p + "report"] = np.asarray([rep.tree_build_bitops, rep.hidft_adds, rep.hidft_mults, rep.solve_adds,
                                        rep.solve_mults, rep.read_ops, rep.samples_touched,
                                        rep.escalated_nodes, rep.dense_fallbacks], np.int64)
        out[p + "bounds"] = np.asarray([rep.bound_alg1bnd, rep.bound_hidft])
        out[p + "systems"] = np.asarray([[s.residue, s.size, int(s.escalated), int(s.dense_fallback)]
                                         for s in res.node_systems], np.int64)
    out["n_cases"] = np.asarray([kept])
    # config 3: the reference's "auto" and "random_subset" policies on
    # signal 0 (dense complex64, as the bench feeds it)
    from structfft.families import rng_from_seed
    piv = tuple(sorted(int(x) for x in rng_from_seed(3, 7).choice(22, size=14, replace=False)))
    H = R.gen_homogeneous(piv, 22, 3)
    pick = np.sort(rng_from_seed(3, 8).choice(1 << 14, size=1 << 12, replace=False))
    J3 = R.SupportSet.make(1 << 22, H.as_array()[pick].tolist())
    g = rng_from_seed(3, 200, 0)
    c3 = g.normal(size=len(J3)) + 1j * g.normal(size=len(J3))
    spec = np.zeros(1 << 22, np.complex128)
    spec[J3.as_array()] = c3
    f3 = np.fft.ifft(spec).astype(np.complex64)
    for pol in ("auto", "random_subset"):
        res = R.sas_transform(f3, J3, policy=pol, family_meta={"base_pivots": piv})
        rep = res.report
        out[f"cfg3_{pol}_coeffs"] = res.coeffs
        out[f"cfg3_{pol}_plan"] = np.asarray([len(res.plan.pivots), res.plan.mu_star, rep.escalated_nodes,
                                              rep.dense_fallbacks, rep.samples_touched], np.int64)
    out["cfg3_base_pivots"] = np.asarray(piv, np.int64)
    np.savez_compressed(os.path.join(HERE, "golden_sas.npz"), **out)
    print("sas cases", kept, "escalations", sum(int(out[f"s{i}_report"][7]) for i in range(kept)))


if __name__ == "__main__":
    main()
