"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `structfft` read-only from /root/reference/pkg/src, evaluates the
hot-path functions on seeded inputs and writes `tests/golden/golden_*.npz`
plus `kats.json`.  The fixtures pin the oracle (oracle/structfft_oracle.py)
and, through it, the CUDA path.  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    import structfft as R
    from structfft.families import rng_from_seed
    from structfft.hidft import _build_plan

    kats: dict = {}

    # ---- pivots / classify / part-homogeneity KATs (tests/test_congruence.py:106-165)
    fixtures = [
        (32, [3, 17, 25, 27]),
        (1024, [23, 187, 190, 247, 386, 731, 990, 994]),
        (1024, [84, 305, 725, 992]),
        (16, [9]),
        (64, [3, 17, 25, 27, 35]),
        (64, [1, 2, 4, 8, 16, 32]),           # J* for M=6 (gen_jstar(6))
        (1024, [316, 384, 828, 896]),
        (8, [0, 1, 3]),
        (1024, [0, 1, 6, 7, 512]),
        (8, [0, 4]),
    ]
    rng = np.random.default_rng(20261020)
    for _ in range(200):
        M = int(rng.integers(2, 14))
        N = 1 << M
        k = int(rng.integers(1, min(N, 64) + 1))
        fixtures.append((N, sorted(rng.choice(N, size=k, replace=False).tolist())))
    piv_cases = []
    for N, idx in fixtures:
        J = R.SupportSet.make(N, idx)
        cls = R.classify(J)
        piv_cases.append({"N": N, "J": list(J.indices), "pivots": list(R.pivots(J)),
                          "kind": cls.kind})
    kats["pivots"] = piv_cases
    kats["part_homogeneous"] = [
        {"N": 64, "J": [3, 17, 25, 27, 35], "r": [1, 3],
         "ok": R.is_part_homogeneous(R.SupportSet.make(64, [3, 17, 25, 27, 35]), (1, 3))},
        {"N": 64, "J": [3, 17, 25, 27, 35], "r": [3],
         "ok": R.is_part_homogeneous(R.SupportSet.make(64, [3, 17, 25, 27, 35]), (3,))},
    ]

    # ---- sample sets I_r (tests/test_sampling.py:27-53)
    pat_cases = [((0, 2), 10), ((), 6), (tuple(range(4)), 4), ((1, 3), 6), ((1, 3), 5),
                 ((0, 2, 5, 9), 12)]
    for _ in range(100):
        M = int(rng.integers(1, 25))
        s = int(rng.integers(0, min(M, 12) + 1))
        pat_cases.append((tuple(sorted(rng.choice(M, size=s, replace=False).tolist())), M))
    kats["patterns"] = [{"r": list(r), "M": M, "I": list(R.pivoted_pattern(r, M).samples)}
                        for r, M in pat_cases]

    with open(os.path.join(HERE, "kats.json"), "w") as fh:
        json.dump(kats, fh, separators=(",", ":"))

    # ---- hidft on dense signals: random homogeneous, part-homogeneous, full support
    cases = []
    for i in range(60):  # tests/test_hidft.py:43-53 shape
        M = int(rng.integers(2, 11))
        s = int(rng.integers(1, min(M, 7) + 1))
        piv = tuple(sorted(rng.choice(M, size=s, replace=False).tolist()))
        J = R.gen_homogeneous(piv, M, int(rng.integers(0, 2 ** 62)))
        n = int(rng.integers(0, s + 1))
        a = int(rng.integers(0, 1 << M))
        cases.append((J, piv, n, a))
    for N, idx, r in [(64, [3, 17, 25, 27, 35], (1, 3)), (1024, [0, 1, 6, 7, 512], (0, 1)),
                      (8, [0, 1, 3], (0, 1)), (32, [3, 17, 25, 27], (1, 3))]:
        J = R.SupportSet.make(N, idx)
        for n in range(len(r) + 1):
            for a in (0, 1, 5):
                cases.append((J, r, n, a))
    for M in (1, 2, 5, 8):  # J = Z_N degenerates to the radix-2 FFT
        cases.append((R.SupportSet.make(1 << M, range(1 << M)), tuple(range(M)), 0, 0))
    out: dict[str, np.ndarray] = {}
    for i, (J, r, n, a) in enumerate(cases):
        N = J.N
        f = rng.normal(size=N) + 1j * rng.normal(size=N)
        res = R.hidft(f, J, r, height=n, shift=a)
        used = r[: len(r) - n]
        plan = _build_plan(J, used)
        p = f"c{i}_"
        out[p + "meta"] = np.asarray([N, n, a, res.level, res.ops_adds, res.ops_mults], np.int64)
        out[p + "J"] = J.as_array()
        out[p + "r"] = np.asarray(r, np.int64)
        out[p + "f"] = f
        out[p + "node_residues"] = np.asarray(res.node_residues, np.int64)
        out[p + "node_values"] = res.node_values
        out[p + "slot_values"] = res.slot_values
        out[p + "slot_residues"] = np.asarray(res.slot_residues, np.int64)
        out[p + "slot_real"] = np.asarray(res.slot_real, bool)
        out[p + "element_slots"] = np.asarray(plan.element_slots, np.int64)
        out[p + "twiddles"] = (np.concatenate(plan.twiddles) if plan.twiddles
                               else np.zeros(0, np.complex128))
        if R.classify(J).is_homogeneous:
            out[p + "dft"] = R.hidft_to_dft(R.hidft(f, J, R.pivots(J)))
    out["n_cases"] = np.asarray([len(cases)])
    np.savez_compressed(os.path.join(HERE, "golden_hidft.npz"), **out)

    # ---- BASELINE configs: supports from the SURVEY 8(d) recipe via the
    # reference generators, and reference outputs on numpy-synthesised signals
    cfg: dict[str, np.ndarray] = {}

    def homog(c, P_hi, p, M):
        piv = sorted(int(x) for x in rng_from_seed(c, 7).choice(P_hi, size=p, replace=False))
        return R.gen_homogeneous(piv, M, c)

    supports = {1: (homog(1, 16, 8, 16), 16), 2: (homog(2, 16, 10, 20), 20),
                5: (homog(5, 26, 16, 26), 26)}
    H = homog(3, 22, 14, 22)
    pick = np.sort(rng_from_seed(3, 8).choice(1 << 14, size=1 << 12, replace=False))
    supports[3] = (R.SupportSet.make(1 << 22, H.as_array()[pick].tolist()), 22)
    for c, (J, M) in supports.items():
        cfg[f"cfg{c}_J"] = J.as_array()
        cfg[f"cfg{c}_pivots"] = np.asarray(R.pivots(J), np.int64)
    h = hashlib.sha256()
    for b in range(256):
        piv = sorted(int(x) for x in rng_from_seed(4, 9, b).choice(16, size=10, replace=False))
        seed_b = int(rng_from_seed(4, 10, b).integers(0, 2 ** 62))
        J = R.gen_homogeneous(piv, 20, seed_b)
        if b < 8:
            cfg[f"cfg4_J{b}"] = J.as_array()
        h.update(J.as_array().astype("<i8").tobytes())
    cfg["cfg4_sha256_first256"] = np.frombuffer(h.digest(), np.uint8)

    dtypes = {1: np.complex128, 2: np.complex64, 3: np.complex64, 5: np.complex64}
    for c, (J, M) in supports.items():
        nsig = 1 if c == 5 else 2
        for b in range(nsig):
            coef = rng_from_seed(c, 200, b)
            coef = coef.normal(size=len(J)) + 1j * coef.normal(size=len(J))
            spec = np.zeros(1 << M, np.complex128)
            spec[J.as_array()] = coef
            f = np.fft.ifft(spec).astype(dtypes[c])
            if c == 3:
                got = R.sas_transform(f, J, r=R.pivots(J)).coeffs
            else:
                got = R.hidft_to_dft(R.hidft(f, J, R.pivots(J)))
            if c == 5:
                cfg[f"cfg{c}_b{b}_head"] = got[:4096]
                cfg[f"cfg{c}_b{b}_sum"] = np.asarray([got.sum(), np.linalg.norm(got)])
            else:
                cfg[f"cfg{c}_b{b}_out"] = got
            cfg[f"cfg{c}_b{b}_coef"] = coef
    for b in range(2):  # per-signal supports
        piv = sorted(int(x) for x in rng_from_seed(4, 9, b).choice(16, size=10, replace=False))
        seed_b = int(rng_from_seed(4, 10, b).integers(0, 2 ** 62))
        J = R.gen_homogeneous(piv, 20, seed_b)
        coef = rng_from_seed(4, 200, b)
        coef = coef.normal(size=len(J)) + 1j * coef.normal(size=len(J))
        spec = np.zeros(1 << 20, np.complex128)
        spec[J.as_array()] = coef
        f = np.fft.ifft(spec).astype(np.complex64)
        cfg[f"cfg4_b{b}_out"] = R.hidft_to_dft(R.hidft(f, J, R.pivots(J)))
        cfg[f"cfg4_b{b}_coef"] = coef
    np.savez_compressed(os.path.join(HERE, "golden_configs.npz"), **cfg)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
