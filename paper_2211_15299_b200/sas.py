"""Shift-and-sample on the device, mu* = 1 path (reference sas.py:313-409).

With the pivot vector chosen so that every node at the decode level r_max+1
holds one element (always true for r = pivots(J)), SAS is a single Hi-DFT
whose node values times N/|I| are the coefficients (sas.py:358-371).  That
is config 3's reference call, `sas_transform(f, J, r=pivots(J))`.  Nodes of
weight > 1 need per-node Vandermonde decoding (sas.py:372-398), which is the
next component on the roadmap and raises
NotImplementedError here rather than silently falling back to the CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .congruence import SupportSet, as_support, pivots as support_pivots, validate_pivot_vector
from .errors import InvalidInputError
from .hidft import _count, _finish, _gathered_samples, _prepare_source, _torch, get_plan

C1 = 1.5  # per-stage butterfly constant (sas.py:38)
C2 = 6.0  # Vandermonde constant (sas.py:39)
POLICIES = ("balanced", "uoe", "uoh", "random_subset", "auto")


def predicted_cost(size_r: int, mu_star: int, node_weights: Sequence[int]) -> float:
    """c1 s 2^s mu* + c2 sum w^2 (sas.py:53-54)."""
    return C1 * size_r * (1 << size_r) * mu_star + C2 * sum(int(w) * int(w) for w in node_weights)


def _weights_at(J: SupportSet, level: int) -> np.ndarray:
    """Node weights of the congruence tree at `level` (counts per residue)."""
    _, counts = np.unique(J.as_array() & ((1 << level) - 1), return_counts=True)
    return counts


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
        p = support_pivots(J)
        best, best_cost = (), math.inf
        for t in range(len(p) + 1):
            level = p[t - 1] + 1 if t else 0
            w = _weights_at(J, level)
            cost = predicted_cost(t, int(w.max()), w)
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


@dataclass
class SasReport:
    hidft_adds: int = 0
    hidft_mults: int = 0
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
    def total(self) -> int:
        return self.ops_hidft + self.read_ops


@dataclass
class SasResult:
    support: SupportSet
    coeffs: object
    plan: SasPlan
    report: SasReport = field(default_factory=SasReport)

    def coeff_map(self) -> dict[int, complex]:
        c = self.coeffs.detach().cpu().numpy() if hasattr(self.coeffs, "detach") else self.coeffs
        return {int(j): complex(v) for j, v in zip(self.support.indices, c)}


def sas_transform(source, J, r: Sequence[int] | None = None, policy: str = "auto",
                  family_meta: dict | None = None, counter=None, tolerance: float = 1e-8) -> SasResult:
    """Recover (F f)_J by shift-and-sample; mu* = 1 only (see module doc)."""
    torch = _torch()
    J = as_support(J)
    rt = select_pivots(J, policy, family_meta) if r is None else validate_pivot_vector(r, J.M)
    src = _prepare_source(source, J.N)
    plan = get_plan(J, rt, 0, src.dtype_code, src.device)
    if plan.mu_star != 1:
        raise NotImplementedError(
            f"mu*={plan.mu_star} > 1 needs per-node Vandermonde decoding (sas.py:372-398), "
            "not on the device path yet; use r=pivots(J)")
    cdt = torch.complex64 if src.dtype_code == _lib.C64 else torch.complex128
    stream = _lib.stream_ptr(src.device)
    if src.kind in ("callable", "synth"):
        samples = _gathered_samples(src, plan, 0)
        out = torch.empty((1, len(J)), dtype=cdt, device=src.device)
        _lib.check(_lib.load().sfft_hidft_gathered(plan.handle, samples.data_ptr(), 1, plan.A, _lib.OUT_SAS,
                                                   out.data_ptr(), len(J), None, 0, stream))
    else:
        sig = src.tensor
        B = sig.shape[0]
        out = torch.empty((B, len(J)), dtype=cdt, device=src.device)
        _lib.check(_lib.load().sfft_hidft(plan.handle, sig.data_ptr(), B, sig.stride(0), 0, _lib.OUT_SAS,
                                          out.data_ptr(), len(J), None, 0, stream))
    _count(counter, plan.A, plan.s)
    scale = J.N / plan.A
    if counter is not None and scale != 1.0:
        counter.mul(len(J), phase="read")
    weights = tuple([1] * plan.n_nodes)
    splan = SasPlan(rt, plan.level, 1, weights, predicted_cost(len(rt), 1, weights))
    rep = SasReport(hidft_adds=plan.A * plan.s, hidft_mults=(plan.A // 2) * plan.s,
                    read_ops=len(J) if scale != 1.0 else 0, samples_touched=plan.A,
                    bound_alg1bnd=splan.predicted_cost, bound_hidft=C1 * len(rt) * (1 << len(rt)))
    return SasResult(J, _finish(out, src), splan, rep)
