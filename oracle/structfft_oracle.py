"""CPU oracle for the Hi-DFT hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `structfft` package's
hot path (arXiv 2211.15299, /root/reference/pkg/src/structfft).  It exists to
CHECK the B200 CUDA path; it is never called by the product code.  Only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import it.

Parity is PINNED: `tests/test_oracle_golden.py` checks every function here
against golden vectors produced by the reference itself
(`tests/golden/make_golden.py`, run in the build container where
/root/reference exists) and against the reference's own known-answer tests
(SURVEY.md section 8(c)).

Conventions (reference core.py:3-6): forward kernel e^{-2 pi i mn/N}; the
shifted signal tau^a f(n) = f(n - a) is read at (I - a) mod N; `hidft`
returns the UNSCALED product F(J, I) f_I and `hidft_to_dft` multiplies by
N/|J| (hidft.py:188-207).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# status codes shared with the C-ABI (errors.py:4-17, cli.py:366-378)
OK, INVALID, CONTRACT, BUDGET = 0, 2, 3, 4


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# ---------------------------------------------------------------- seeding ---

def rng_from_seed(seed: int, *streams: int) -> np.random.Generator:
    """Counter-based Philox stream keyed by (seed, streams); families.py:35-37."""
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(int(s) for s in streams))
    return np.random.Generator(np.random.Philox(seed=ss))


def gen_homogeneous(r, M: int, seed: int) -> np.ndarray:
    """Homogeneous support with pivot vector r; families.py:61-80.

    J = {a + sum_i b_i c_i 2^{r_i} mod N : b in {0,1}^s}; a uniform in [0, N),
    c_i odd in [1, 2^{M-r_i}).  Draw order (a first, then one draw per pivot)
    matches the reference so that the same seed yields the same set.
    """
    r = validate_pivot_vector(r, M)
    N = 1 << M
    rng = rng_from_seed(seed, 1)
    a = int(rng.integers(0, N))
    mults = [1 + 2 * int(rng.integers(0, max(1 << (M - ri - 1), 1))) for ri in r]
    vals = np.asarray([a], dtype=np.int64)
    for c, ri in zip(mults, r):
        vals = np.concatenate([vals, (vals + (c << ri)) % N])
    J = np.unique(vals % N)
    if pivots(J, M) != r:
        raise OracleError(CONTRACT, "homogeneous construction missed its pivots")
    return J


def complex_gaussian(k: int, rng: np.random.Generator) -> np.ndarray:
    """families.py:48 (draw_coefficients, nonzero=False)."""
    return rng.normal(size=k) + 1j * rng.normal(size=k)


# ------------------------------------------------------------ congruence ---

def validate_support(J, N: int) -> np.ndarray:
    """SupportSet invariants (congruence.py:41-50)."""
    if N <= 0 or N & (N - 1):
        raise OracleError(INVALID, f"N={N} is not a power of two")
    arr = np.asarray(J, dtype=np.int64).reshape(-1)
    if arr.size == 0:
        raise OracleError(INVALID, "support set is empty")
    if (arr < 0).any() or (arr >= N).any():
        raise OracleError(INVALID, "support indices must lie in [0, N)")
    if arr.size > 1 and (np.diff(arr) <= 0).any():
        raise OracleError(INVALID, "support indices must be strictly increasing")
    return arr


def validate_pivot_vector(r, M: int) -> tuple[int, ...]:
    """congruence.py:272-278."""
    rt = tuple(int(x) for x in r)
    if any(a >= b for a, b in zip(rt, rt[1:])):
        raise OracleError(INVALID, "pivot vector must be strictly increasing")
    if any(x < 0 or x >= M for x in rt):
        raise OracleError(INVALID, f"pivots must lie in [0, {M})")
    return rt


def pivots(J, M: int) -> tuple[int, ...]:
    """Split levels of the congruence tree; congruence.py:76-101.

    Level l splits iff the number of distinct residues mod 2^{l+1} exceeds
    the number mod 2^l (partition refinement by residue class), stopping once
    every class is a singleton.
    """
    arr = np.asarray(J, dtype=np.int64)
    k = arr.size
    out = []
    prev = 1
    for level in range(M):
        if prev == k:
            break
        cnt = np.unique(arr & ((1 << (level + 1)) - 1)).size
        if cnt > prev:
            out.append(level)
        prev = cnt
    return tuple(out)


def pivots_pairwise(J) -> tuple[int, ...]:
    """{v2(j1 - j2)} by definition (congruence.py:104-120); small sets only."""
    arr = np.asarray(J, dtype=np.int64)
    x = arr[:, None] ^ arr[None, :]
    x = x[x != 0]
    low = x & -x
    return tuple(sorted({int(v).bit_length() - 1 for v in np.unique(low)}))


def is_homogeneous(J, M: int) -> bool:
    """classify(J).is_homogeneous; congruence.py:235-241."""
    k = len(J)
    return k & (k - 1) == 0 and len(pivots(J, M)) == k.bit_length() - 1


def part_homogeneity_violation(J, M: int, r) -> int | None:
    """First pivot <= max(r) missing from r, or None; congruence.py:259-269."""
    r = tuple(r)
    if not r:
        return None
    rmax, rs = max(r), set(r)
    for p in pivots(J, M):
        if p <= rmax and p not in rs:
            return p
    return None


# ---------------------------------------------------------------- sampling ---

def pivoted_pattern(r, M: int) -> np.ndarray:
    """I_r = sorted {sum_i b_i 2^{M-1-r_i}}; sampling.py:47-71."""
    r = validate_pivot_vector(r, M)
    vals = np.zeros(1, dtype=np.int64)
    for ri in r:
        vals = np.concatenate([vals, vals + (1 << (M - 1 - ri))])
    out = np.sort(vals)
    if np.unique(out).size != out.size:
        raise OracleError(INVALID, "pattern elements are not distinct")
    return out


def slot_offsets(used, M: int) -> np.ndarray:
    """Gather offsets in slot order; hidft.py:155-158."""
    A = 1 << len(used)
    a = np.arange(A, dtype=np.int64)
    off = np.zeros(A, dtype=np.int64)
    for i, rk in enumerate(used):
        off += ((a >> i) & 1) << (M - 1 - rk)
    return off


# ------------------------------------------------------------------- plan ---

@dataclass
class Plan:
    used: tuple[int, ...]
    level: int
    element_slots: np.ndarray   # (k,) slot of each support element
    slot_residues: np.ndarray   # (A,) residue mod 2^level (virtual slots inherit)
    slot_real: np.ndarray       # (A,) bool
    slot_count: np.ndarray      # (A,) members per slot (node weight)
    twiddles: list              # stage k: 2^(k-1) complex128
    offsets: np.ndarray         # (A,) gather offsets, slot order
    node_slots: np.ndarray      # real slots in ascending residue order
    node_residues: np.ndarray

    @property
    def A(self) -> int:
        return 1 << len(self.used)


def build_plan(J, M: int, used) -> Plan:
    """Restates hidft._build_plan (hidft.py:69-95) plus offsets / node order.

    Per stage k (merging pivot used[k-1]) the least member of every slot
    prefix becomes its representative; empty prefixes ("virtual" slots)
    inherit the parent's residue below used[k-1] with the branch bit set.
    """
    arr = np.asarray(J, dtype=np.int64)
    s = len(used)
    A = 1 << s
    pats = np.zeros(arr.size, dtype=np.int64)
    for i, rk in enumerate(used):
        pats |= ((arr >> rk) & 1) << i
    reps = np.array([arr.min()], dtype=np.int64)
    twiddles = []
    empty = np.iinfo(np.int64).max
    for k, rk in enumerate(used, start=1):
        shared = reps & ((1 << rk) - 1)
        twiddles.append(np.exp(-2j * np.pi * (shared + (1 << rk)) / float(1 << (rk + 1))))
        width = 1 << k
        mins = np.full(width, empty, dtype=np.int64)
        np.minimum.at(mins, pats & (width - 1), arr)
        idx = np.arange(width)
        inherit = shared[idx & ((width >> 1) - 1)] + (((idx >> (k - 1)) & 1) << rk)
        reps = np.where(mins == empty, inherit, mins)
    level = used[-1] + 1 if s else 0
    slot_res = reps & ((1 << level) - 1)
    count = np.bincount(pats, minlength=A)
    real = count > 0
    real_slots = np.nonzero(real)[0]
    order = np.argsort(slot_res[real_slots], kind="stable")
    return Plan(tuple(used), level, pats, slot_res, real, count, twiddles,
                slot_offsets(used, M), real_slots[order], slot_res[real_slots][order])


def butterfly(v: np.ndarray, plan: Plan) -> np.ndarray:
    """Generalised radix-2 stages over the last axis; hidft.py:160-167.

    Stage k pairs slots differing in bit k-1: branch 0 = v0 - w v1,
    branch 1 = v0 + w v1 with w = twiddles[k-1][low k-1 slot bits].
    Works on (A,) or (B, A) complex128.
    """
    lead = v.shape[:-1]
    A = v.shape[-1]
    for k in range(1, len(plan.used) + 1):
        half = 1 << (k - 1)
        x = v.reshape(lead + (A // (2 * half), 2, half))
        t = plan.twiddles[k - 1][None, :] * x[..., 1, :]
        v = np.stack([x[..., 0, :] - t, x[..., 0, :] + t], axis=-2).reshape(lead + (A,))
    return v


@dataclass
class HiDftOut:
    level: int
    node_residues: np.ndarray
    node_values: np.ndarray      # (..., n_nodes)
    slot_values: np.ndarray      # (..., A)
    slot_residues: np.ndarray
    slot_real: np.ndarray
    ops_adds: int
    ops_mults: int


def hidft(signals, J, M: int, r, height: int = 0, shift: int = 0) -> HiDftOut:
    """hidft.py:135-185 on dense signals (N,) or (B, N), any complex dtype.

    Samples are promoted to complex128 exactly as the reference does
    (hidft.py:46), then the butterfly runs in float64.
    """
    rt = validate_pivot_vector(r, M)
    bad = part_homogeneity_violation(J, M, rt)
    if bad is not None:
        raise OracleError(CONTRACT, f"support is not {rt}-part-homogeneous: pivot {bad}")
    if height < 0 or height > len(rt):
        raise OracleError(INVALID, f"height must be in [0, {len(rt)}]")
    used = rt[: len(rt) - height]
    plan = build_plan(J, M, used)
    N = 1 << M
    loc = (plan.offsets - shift) % N
    sig = np.asarray(signals)
    v = sig[..., loc].astype(np.complex128)
    v = butterfly(v, plan)
    s = len(used)
    return HiDftOut(plan.level, plan.node_residues, v[..., plan.node_slots], v,
                    plan.slot_residues, plan.slot_real, plan.A * s, (plan.A // 2) * s)


def hidft_to_dft(signals, J, M: int) -> np.ndarray:
    """hidft(f, J, pivots(J)) followed by hidft_to_dft (hidft.py:188-207).

    Output in ascending-J order, scaled by N/k (skipped when N/k == 1).
    """
    if not is_homogeneous(J, M):
        raise OracleError(CONTRACT, "hidft_to_dft requires a homogeneous support")
    r = pivots(J, M)
    plan = build_plan(J, M, r)
    N = 1 << M
    sig = np.asarray(signals)
    v = butterfly(sig[..., plan.offsets % N].astype(np.complex128), plan)
    vals = v[..., plan.element_slots]
    factor = N / len(J)
    return vals if factor == 1.0 else vals * factor


def sas_mu1(signals, J, M: int, r=None) -> np.ndarray:
    """sas_transform's mu*=1 path (sas.py:313-371,400-409).

    With r = pivots(J) (default) every node at level r_max+1 is a singleton;
    the coefficient of j is its node value times N/|I|, ascending-J order.
    """
    rt = pivots(J, M) if r is None else validate_pivot_vector(r, M)
    bad = part_homogeneity_violation(J, M, rt)
    if bad is not None:
        raise OracleError(CONTRACT, f"not part-homogeneous: pivot {bad}")
    plan = build_plan(J, M, rt)
    if plan.slot_count.max() != 1:
        raise OracleError(CONTRACT, "mu* > 1: Vandermonde decoding required")
    N = 1 << M
    sig = np.asarray(signals)
    v = butterfly(sig[..., plan.offsets % N].astype(np.complex128), plan)
    vals = v[..., plan.element_slots]
    scale = N / plan.A
    return vals if scale == 1.0 else vals * scale


def dense_submatrix(signal, J, M: int, r, height: int = 0, shift: int = 0) -> np.ndarray:
    """F(node reps, I) f_I by definition (hidft.py:210-237, core.py:193-215)."""
    rt = validate_pivot_vector(r, M)
    used = rt[: len(rt) - height]
    level = used[-1] + 1 if used else 0
    N = 1 << M
    cols = pivoted_pattern(used, M)
    f = np.asarray(signal, dtype=np.complex128)[(cols - shift) % N]
    reps = np.unique(np.asarray(J, dtype=np.int64) & ((1 << level) - 1))
    kern = np.exp(-2j * np.pi * ((np.outer(reps, cols) % N) / N))
    return kern @ f


# ----------------------------------------------------- reference-shaped path ---

def reference_call(signal, J, M: int) -> np.ndarray:
    """One reference public call, cost-faithful: hidft(f, J, pivots(J)) then
    hidft_to_dft (hidft.py:135-207).  Pivots are re-derived three times and
    the dense input is promoted whole to complex128, as the reference does;
    used as the CPU baseline leg of bench.py."""
    r = pivots(J, M)                                      # caller's pivots(J)
    validate_pivot_vector(r, M)
    if part_homogeneity_violation(J, M, r) is not None:   # assert_part_homogeneous
        raise OracleError(CONTRACT, "not part-homogeneous")
    plan = build_plan(J, M, r)
    N = 1 << M
    arr = np.asarray(signal, dtype=np.complex128)         # whole-array upcast
    v = butterfly(arr[plan.offsets % N], plan)
    node_vals = v[plan.node_slots]
    if not is_homogeneous(J, M):                          # classify in hidft_to_dft
        raise OracleError(CONTRACT, "hidft_to_dft requires a homogeneous support")
    values = {int(res): complex(x) for res, x in zip(plan.node_residues, node_vals)}
    mask = (1 << plan.level) - 1
    out = np.asarray([values[int(j) & mask] for j in J], dtype=np.complex128)
    factor = N / len(J)
    return out if factor == 1.0 else out * factor


def reference_sas_call(signal, J, M: int) -> np.ndarray:
    """Cost-faithful sas_transform(f, J, r=pivots(J)) mu*=1 call (sas.py:313-409)."""
    r = pivots(J, M)
    if part_homogeneity_violation(J, M, r) is not None:
        raise OracleError(CONTRACT, "not part-homogeneous")
    plan = build_plan(J, M, r)
    N = 1 << M
    pattern = pivoted_pattern(r, M)
    arr = np.asarray(signal, dtype=np.complex128)
    v = butterfly(arr[plan.offsets % N], plan)
    values = {int(res): complex(x) for res, x in zip(plan.node_residues, v[plan.node_slots])}
    mask = (1 << plan.level) - 1
    scale = N / pattern.size
    return np.asarray([values[int(j) & mask] * scale for j in J], dtype=np.complex128)


# --------------------------------------------------------------- configs ---

def config_support(cfg: int, b: int = 0):
    """Support(s) for BASELINE.json configs, SURVEY.md section 8(d) recipe.

    Returns (J int64 array, M).  cfg4 draws one support per signal b.
    """
    if cfg in (1, 2, 5):
        P_hi, p, M = {1: (16, 8, 16), 2: (16, 10, 20), 5: (26, 16, 26)}[cfg]
        piv = sorted(int(x) for x in rng_from_seed(cfg, 7).choice(P_hi, size=p, replace=False))
        return gen_homogeneous(piv, M, cfg), M
    if cfg == 3:
        M = 22
        piv = sorted(int(x) for x in rng_from_seed(3, 7).choice(22, size=14, replace=False))
        H = gen_homogeneous(piv, M, 3)
        pick = np.sort(rng_from_seed(3, 8).choice(1 << 14, size=1 << 12, replace=False))
        return H[pick], M
    if cfg == 4:
        M = 20
        piv = sorted(int(x) for x in rng_from_seed(4, 9, b).choice(16, size=10, replace=False))
        seed_b = int(rng_from_seed(4, 10, b).integers(0, 2 ** 62))
        return gen_homogeneous(piv, M, seed_b), M
    raise ValueError(f"unknown config {cfg}")


def config_coefficients(cfg: int, b: int, k: int) -> np.ndarray:
    """Coefficients of signal b: rng_from_seed(cfg, 200, b) complex Gaussian."""
    return complex_gaussian(k, rng_from_seed(cfg, 200, b))


def synthesize(J, coeffs, M: int) -> np.ndarray:
    """f = ifft of the zero-padded spectrum (1/N scaling; core.py:3-6), c128."""
    N = 1 << M
    spec = np.zeros(N, dtype=np.complex128)
    spec[np.asarray(J, dtype=np.int64)] = coeffs
    return np.fft.ifft(spec)

