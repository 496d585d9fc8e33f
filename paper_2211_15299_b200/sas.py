"""Shift-and-sample on the device (reference sas.py:313-409).

The transform picks a pivot vector r with J r-part-homogeneous (the
reference's policies, sas.py:89-129), computes the Hi-DFT of tau^j f for
j < mu* (mu* = largest node weight at the decode level r_max+1) as ONE
launch over B*mu* rows, and decodes each aliased node v from
(N/|I|) Hidft(tau^j f)(v) = sum_{l in v} Ff(l) x_l^j, x_l = e^{-2 pi i l/N}:
Bjorck-Pereyra with Leja order in float64, the reference's forward-error
estimate, double-double re-measure and re-solve above tolerance/20 and a
dense LU fallback (sfft_sas_decode).  With mu* = 1 (e.g. r = pivots(J),
config 3) it is a single Hi-DFT read scaled by N/|I| in the input precision.
Node weights up to 64 are decoded one (signal, node) per thread, heavier
nodes (up to 1024) one per CTA with their arrays in shared memory.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .congruence import (SupportSet, as_support, assert_part_homogeneous, pivots as support_pivots,
                         validate_pivot_vector)
from .errors import InvalidInputError
from .hidft import (_finish, _gathered_samples, _host_threads, _host_transform, _prepare_source, _torch,
                    get_plan)

C1 = 1.5  # per-stage butterfly constant (sas.py:38)
C2 = 6.0  # Vandermonde constant (sas.py:39)
POLICIES = ("balanced", "uoe", "uoh", "random_subset", "auto")


def predicted_cost(size_r: int, mu_star: int, node_weights: Sequence[int]) -> float:
    """c1 s 2^s mu* + c2 sum w^2 (sas.py:53-54)."""
    return C1 * size_r * (1 << size_r) * mu_star + C2 * sum(int(w) * int(w) for w in node_weights)


def _prefix_profile(J: SupportSet, piv: tuple[int, ...]) -> tuple[np.ndarray, np.ndarray]:
    """(mu*, sum w^2) at the decode level of every prefix of piv (sfft_prefix_weights),
    cached on the immutable support."""
    key = ("prefix_profile", tuple(piv))
    if key in J._plans:
        return J._plans[key]
    dev = _lib.require_device()
    s = len(piv)
    mu = np.zeros(s + 1, np.uint64)
    sq = np.zeros(s + 1, np.uint64)
    pv = np.asarray(piv if piv else [0], np.int32)
    _lib.check(_lib.load().sfft_prefix_weights(J.device_tensor(dev).data_ptr(), len(J), J.M, pv.ctypes.data, s,
                                               mu.ctypes.data, sq.ctypes.data, _lib.stream_ptr(dev)))
    J._plans[key] = (mu.astype(np.int64), sq.astype(np.int64))
    return J._plans[key]


def _stock_pivot_count(k: int) -> int:
    """floor(log2 k - log2 log2 k); k < 3 -> k - 1 (sas.py:46-50)."""
    if k < 3:
        return max(k - 1, 0)
    return max(int(math.floor(math.log2(k) - math.log2(math.log2(k)))), 0)


def select_pivots(J, policy: str = "auto", family_meta: dict | None = None) -> tuple[int, ...]:
    """Pivot-vector policies of sas.py:89-129 (planning on the support only)."""
    J = as_support(J)
    if policy not in POLICIES:
        raise InvalidInputError(f"unknown policy {policy!r}; expected one of {POLICIES}")
    meta = family_meta or {}
    if policy == "auto":
        # node-weight profile of every prefix of pivots(J), one device pass
        p = support_pivots(J)
        mu, sq = _prefix_profile(J, p)
        best, best_cost = (), math.inf
        for t in range(len(p) + 1):
            cost = C1 * t * (1 << t) * mu[t] + C2 * sq[t]
            if cost < best_cost:  # ties keep the shorter prefix
                best, best_cost = p[:t], cost
        r = best
    elif policy == "balanced":
        if "pivots" not in meta:
            raise InvalidInputError("balanced policy needs family_meta['pivots']")
        r = tuple(int(x) for x in meta["pivots"])
    elif policy == "uoe":
        r = tuple(range(min(_stock_pivot_count(len(J)), J.M)))
    else:
        if "base_pivots" not in meta:
            raise InvalidInputError(f"{policy} policy needs family_meta['base_pivots']")
        base = tuple(int(x) for x in meta["base_pivots"])
        r = base[: min(_stock_pivot_count(len(J)), len(base))]
    rt = validate_pivot_vector(r, J.M)
    from .congruence import assert_part_homogeneous
    assert_part_homogeneous(J, rt)
    return rt


@dataclass(frozen=True)
class SasPlan:
    pivots: tuple[int, ...]
    decode_level: int
    mu_star: int
    node_weights: tuple[int, ...]
    predicted_cost: float

    @property
    def shifts(self) -> range:
        return range(self.mu_star)

    @classmethod
    def plan(cls, J, r: Sequence[int], counter=None) -> "SasPlan":
        """sas.py:69-77: validate r, require r-part-homogeneity, take the node
        weights of T(J) at the decode level r_max+1 (one level of the device
        tree, sfft_tree_build; the counter is charged the reference's
        build_tree cost |J| * level)."""
        from .congruence import level_weights
        J = as_support(J)
        rt = validate_pivot_vector(r, J.M)
        assert_part_homogeneous(J, rt)
        level = rt[-1] + 1 if rt else 0
        if counter is not None:
            counter.count_bit_ops(len(J) * max(level, 1))
        weights = tuple(int(w) for w in level_weights(J, level))
        mu = max(weights)
        return cls(rt, level, mu, weights, predicted_cost(len(rt), mu, weights))


@dataclass
class CostReport:
    """Per-phase costs of one transform run plus the analytic bounds
    (reference counting.py:83-150)."""

    tree_build_bitops: int = 0
    hidft_adds: int = 0
    hidft_mults: int = 0
    solve_adds: int = 0
    solve_mults: int = 0
    read_ops: int = 0
    samples_touched: int = 0
    bound_alg1bnd: float = 0.0
    bound_hidft: float = 0.0
    escalated_nodes: int = 0
    dense_fallbacks: int = 0

    @property
    def ops_hidft(self) -> int:
        return self.hidft_adds + self.hidft_mults

    @property
    def ops_solve(self) -> int:
        return self.solve_adds + self.solve_mults + self.read_ops

    @property
    def total(self) -> int:
        return self.ops_hidft + self.ops_solve

    @classmethod
    def from_counter(cls, counter, **extra) -> "CostReport":
        ha, hm = counter.phase("hidft")
        sa, sm = counter.phase("solve")
        ra, rm = counter.phase("read")
        return cls(tree_build_bitops=counter.bit_ops, hidft_adds=ha, hidft_mults=hm, solve_adds=sa,
                   solve_mults=sm, read_ops=ra + rm, **extra)

    def as_dict(self) -> dict:
        d = dict(self.__dict__)
        d.update(ops_hidft=self.ops_hidft, ops_solve=self.ops_solve, ops_total=self.total)
        return d


SasReport = CostReport  # round-1 name


@dataclass
class NodeSystem:
    residue: int
    members: tuple[int, ...]
    escalated: bool = False
    dense_fallback: bool = False
    residual: float = 0.0

    @property
    def size(self) -> int:
        return len(self.members)


class SasResult:
    """coeffs, plan, report as the reference (sas.py:251-260); node_systems is
    built on first access (per-node records of the first signal); flags holds
    all signals' (B, n_nodes) escalation / fallback markers (1 / 2)."""

    def __init__(self, support, coeffs, plan, report, systems_fn=None, flags=None):
        self.support = support
        self.coeffs = coeffs
        self.plan = plan
        self.report = report
        self._systems_fn = systems_fn
        self._systems = None
        self.flags = flags

    @property
    def node_systems(self) -> list:
        if self._systems is None:
            self._systems = self._systems_fn() if self._systems_fn else []
        return self._systems

    def coeff_map(self) -> dict[int, complex]:
        c = self.coeffs.detach().cpu().numpy() if hasattr(self.coeffs, "detach") else self.coeffs
        return {int(j): complex(v) for j, v in zip(self.support.indices, c)}


def _sas_static(plan64, J: SupportSet, rt: tuple[int, ...], dev, stream) -> dict:
    """Per-plan constants of sas_transform, computed once and cached on the
    (immutable) plan: node membership CSR, node weights, the SasPlan, the
    samples-touched count and the per-signal solve/read op counts."""
    st = getattr(plan64, "_sas_static", None)
    if st is not None:
        return st
    lib = _lib.load()
    k, mu, N, A = len(J), plan64.mu_star, J.N, plan64.A
    off = np.empty(plan64.n_nodes + 1, np.int32)
    mem = np.empty(k, np.int32)
    _lib.check(lib.sfft_plan_nodes(plan64.handle, off.ctypes.data, mem.ctypes.data, stream))
    w = np.diff(off).astype(np.int64)
    weights = tuple(int(x) for x in w)
    splan = SasPlan(rt, plan64.level, mu, weights, predicted_cost(len(rt), mu, weights))
    from .sampling import pivoted_pattern_tensor
    pat = pivoted_pattern_tensor(rt, J.M, dev).cpu().numpy() if rt else np.zeros(1, np.int64)
    single, multi = w == 1, w >= 2
    half = w * (w - 1) // 2
    st = {"off": off, "mem": mem, "w": w, "splan": splan, "touched": _samples_touched(pat, mu, N),
          "read_mul": int(single.sum()) if N != A else 0,
          "solve_mul": (int(w[multi].sum()) if N != A else 0) + int((w * (w - 1))[multi].sum() + half[w >= 3].sum()),
          "solve_add": int((3 * half)[multi].sum() + half[w >= 3].sum())}
    plan64._sas_static = st
    plan64._nodes = (off, mem)
    return st


def _samples_touched(pattern: np.ndarray, mu: int, N: int) -> int:
    """|union_{j < mu} (I - j) mod N| from the sorted pattern's circular gaps."""
    if pattern.size == 1:
        return min(mu, N)
    gaps = np.diff(np.concatenate([pattern[-1:] - N, pattern]))
    return int(np.minimum(gaps, mu).sum())


def sas_transform(source, J, r: Sequence[int] | None = None, policy: str = "auto",
                  family_meta: dict | None = None, counter=None, tolerance: float = 1e-8) -> SasResult:
    """Recover (F f)_J from mu* shifted Hi-DFTs plus per-node Vandermonde
    decodes (sas.py:313-409), all on the device."""
    from .hidft import _device_guard
    with _device_guard(source):
        return _sas_transform(source, J, r, policy, family_meta, counter, tolerance)


def _sas_transform(source, J, r, policy, family_meta, counter, tolerance) -> SasResult:
    import ctypes
    torch = _torch()
    from .counting import OpCounter
    counter = counter if counter is not None else OpCounter()
    J = as_support(J)
    rt = select_pivots(J, policy, family_meta) if r is None else validate_pivot_vector(r, J.M)
    assert_part_homogeneous(J, rt)
    src = _prepare_source(source, J.N)
    dev = src.device
    lib = _lib.load()
    stream = _lib.stream_ptr(dev)
    plan64 = get_plan(J, rt, 0, _lib.C128, dev)
    mu, level, A, N, k = plan64.mu_star, plan64.level, plan64.A, J.N, len(J)
    scale = N / A
    st = _sas_static(plan64, J, rt, dev, stream)
    off, mem, splan = st["off"], st["mem"], st["splan"]
    counter.count_bit_ops(k * max(level, 1))  # build_tree(J, level) as SasPlan.plan does
    B = 1 if src.kind in ("callable", "synth") else src.tensor.shape[0]
    nn = plan64.n_nodes
    flags = None
    if mu == 1:
        plan = get_plan(J, rt, 0, src.dtype_code, dev)
        cdt = torch.complex64 if src.dtype_code == _lib.C64 else torch.complex128
        if src.kind in ("callable", "synth"):
            samples = _gathered_samples(src, plan, 0)
            out = torch.empty((1, k), dtype=cdt, device=dev)
            _lib.check(lib.sfft_hidft_gathered(plan.handle, samples.data_ptr(), 1, plan.A, _lib.OUT_SAS,
                                               out.data_ptr(), k, None, 0, stream))
        elif src.kind == "host":  # host rows: host gather of the 2^s samples, pipelined DMA
            out = _host_transform(src.tensor, plan, 0, _lib.OUT_SAS, k)
        else:
            sig = src.tensor
            out = torch.empty((B, k), dtype=cdt, device=dev)
            _lib.check(lib.sfft_hidft(plan.handle, sig.data_ptr(), B, sig.stride(0), 0, _lib.OUT_SAS,
                                      out.data_ptr(), k, None, 0, stream))
        n_esc = n_fb = 0
        resid_h = flags_h = None
    else:
        if mu > 1024:
            raise NotImplementedError(f"node weight mu*={mu} above the device decoder's 1024")
        nodevals = torch.empty((B * mu, nn), dtype=torch.complex128, device=dev)
        sig_ptr, ld_sig, sig_dt, table, blJ, blc, ksrc = None, 0, 0, None, None, None, 0
        if src.kind in ("callable", "synth"):
            samples = torch.cat([_gathered_samples(src, plan64, j) for j in range(mu)], 0)
            _lib.check(lib.sfft_hidft_gathered(plan64.handle, samples.data_ptr(), mu, A, _lib.OUT_NODES,
                                               nodevals.data_ptr(), nn, None, 0, stream))
            if src.kind == "synth":
                blJ_t, blc_t = src.fn._device(dev)
                blJ, blc, ksrc = blJ_t.data_ptr(), blc_t.data_ptr(), blJ_t.numel()
            else:  # float64 samples in pattern order for the double-double re-measure
                from .sampling import pivoted_pattern_tensor
                pat = pivoted_pattern_tensor(rt, J.M, dev).cpu().numpy()
                locs = (pat[None, :] - np.arange(mu)[:, None]) % N
                vals = np.asarray(src.fn(locs.reshape(-1)), dtype=np.complex128).reshape(mu, A)
                table_t = torch.from_numpy(vals).to(dev)
                table = table_t.data_ptr()
        elif src.kind == "host":
            # host rows: the host pool stages the mu* shifted sample sets per
            # signal (pattern order, promoted to complex128) on the device;
            # they feed the shifted transforms and the escalation re-measure
            sig = src.tensor
            table_t = torch.empty((B * mu, A), dtype=torch.complex128, device=dev)
            _lib.check(lib.sfft_host_stage(plan64.handle, sig.data_ptr(), B, sig.stride(0), src.dtype_code, 0, mu,
                                           _lib.ORDER_PATTERN, _lib.C128, table_t.data_ptr(), A,
                                           _host_threads(), stream))
            _lib.check(lib.sfft_hidft_staged(plan64.handle, table_t.data_ptr(), B * mu, A, _lib.ORDER_PATTERN,
                                             _lib.OUT_NODES, nodevals.data_ptr(), nn, None, 0, stream))
            table = table_t.data_ptr()
        else:
            sig = src.tensor
            _lib.check(lib.sfft_hidft_shifts(plan64.handle, sig.data_ptr(), B, sig.stride(0), src.dtype_code, 0, mu,
                                             _lib.OUT_NODES, nodevals.data_ptr(), nn, stream))
            sig_ptr, ld_sig, sig_dt = sig.data_ptr(), sig.stride(0), src.dtype_code
        out = torch.empty((B, k), dtype=torch.complex128, device=dev)
        flags = torch.empty((B, nn), dtype=torch.int32, device=dev)
        resid = torch.empty((B, nn), dtype=torch.float64, device=dev)
        ne, nf = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(lib.sfft_sas_decode(plan64.handle, nodevals.data_ptr(), nn, _lib.C128, B, mu, float(tolerance),
                                       sig_ptr, ld_sig, sig_dt, table, blJ, blc, ksrc,
                                       J.device_tensor(dev).data_ptr(), out.data_ptr(), k, flags.data_ptr(),
                                       resid.data_ptr(), ctypes.byref(ne), ctypes.byref(nf), stream))
        n_esc, n_fb = int(ne.value), int(nf.value)
        flags_h, resid_h = flags[0], resid[0]  # device rows, read when node_systems is first used
    # exact counts (sas.py:343-398 with vandermonde_solve's formula, sas.py:196-202)
    if plan64.s:  # mu* shifted Hi-DFTs per signal: A/2 mults + A adds per stage (hidft.py:165-167)
        counter.mul((A // 2) * plan64.s * mu * B, phase="hidft")
        counter.add(A * plan64.s * mu * B, phase="hidft")
    if st["read_mul"]:
        counter.mul(st["read_mul"] * B, phase="read")
    counter.mul(st["solve_mul"] * B, phase="solve")
    counter.add(st["solve_add"] * B, phase="solve")
    if n_fb:
        fb_per_node = (flags.cpu().numpy() == 2).sum(0)
        nfb = int((fb_per_node * st["w"] ** 3).sum())
        counter.mul(nfb, phase="solve")
        counter.add(nfb, phase="solve")
    report = CostReport.from_counter(counter, samples_touched=st["touched"],
                                     bound_alg1bnd=splan.predicted_cost, bound_hidft=C1 * len(rt) * (1 << len(rt)),
                                     escalated_nodes=n_esc, dense_fallbacks=n_fb)

    def systems():
        node_res = plan64.tables()["node_residues"].tolist()
        members = np.split(J._arr[mem], off[1:-1])
        fl = flags_h.cpu().numpy() if flags_h is not None else np.zeros(nn, np.int32)
        rs = resid_h.cpu().numpy() if resid_h is not None else np.zeros(nn)
        return [NodeSystem(node_res[v], tuple(members[v].tolist()), escalated=bool(fl[v] == 1),
                           dense_fallback=bool(fl[v] == 2), residual=float(rs[v])) for v in range(nn)]

    return SasResult(J, _finish(out, src), splan, report, systems, flags)
