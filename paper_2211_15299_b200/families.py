"""Seeded support-family generators (reference families.py:35-353), host side.

These build the supports the CLI's `gen` and `bench` commands and the bench
harness feed to the device transforms.  Every generator draws from the same
Philox streams, in the same order, as the reference, so a (kind, params,
seed) triple yields the same support; the structural claims are re-checked
with the device pivot analysis.  Harness code: nothing here is on the
transform path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .congruence import SupportSet, classify, pivots, validate_pivot_vector
from .errors import ContractViolationError, InvalidInputError
from .workloads import rng_from_seed

KINDS = ("elementary", "homogeneous", "consecutive", "ap", "gap", "uoe", "uoh", "random_subset", "jstar")


def draw_coefficients(k: int, rng, nonzero: bool = True) -> np.ndarray:
    """Nonzero: magnitudes in [0.5, 1.5) with uniform phases; else complex
    Gaussian (families.py:40-48)."""
    if not nonzero:
        return rng.normal(size=k) + 1j * rng.normal(size=k)
    mag = 0.5 + rng.random(k)
    return mag * np.exp(1j * (rng.random(k) * 2 * np.pi))


def _support(N: int, idx) -> SupportSet:
    return SupportSet(N, np.unique(np.fromiter((int(x) for x in idx), dtype=np.int64)))


def elementary(r: int, M: int, seed: int) -> SupportSet:
    """One element per residue class mod 2^r (pivots exactly 0..r-1)."""
    if not 0 <= r <= M:
        raise InvalidInputError("need 0 <= r <= M")
    hi = rng_from_seed(seed, 0).integers(0, 1 << (M - r), size=1 << r)
    return _support(1 << M, (np.arange(1 << r) + (hi << r)) % (1 << M))


def homogeneous(r, M: int, seed: int) -> SupportSet:
    """{a + sum_i b_i c_i 2^{r_i}}: offset a, then one odd c_i per pivot; the
    realised pivots are checked on the device."""
    rt = validate_pivot_vector(r, M)
    N = 1 << M
    g = rng_from_seed(seed, 1)
    a = int(g.integers(0, N))
    vals = np.array([a], dtype=np.int64)
    for ri in rt:
        c = 1 + 2 * int(g.integers(0, max(1 << (M - ri - 1), 1)))
        vals = np.concatenate([vals, (vals + (c << ri)) % N])
    J = _support(N, vals)
    if pivots(J) != rt:
        raise ContractViolationError("homogeneous construction missed its pivots")
    return J


def arithmetic(a: int, s: int, k: int, N: int) -> SupportSet:
    """{a + i s mod N : i < k}, collision-free."""
    if not 1 <= k <= N:
        raise InvalidInputError("need 1 <= k <= N")
    vals = (a + np.arange(k, dtype=np.int64) * s) % N
    if np.unique(vals).size != k:
        raise InvalidInputError("arithmetic progression collides mod N")
    return _support(N, vals)


def generalized_ap(a: int, steps, lengths, N: int) -> tuple[SupportSet, bool]:
    """{a + sum n_i s_i : n_i < N_i} mod N and whether it is proper."""
    steps, lengths = tuple(int(x) for x in steps), tuple(int(x) for x in lengths)
    if len(steps) != len(lengths):
        raise InvalidInputError("steps and lengths must align")
    if not 1 <= len(steps) <= 4:
        raise InvalidInputError("GAP dimension capped at 4")
    if min(lengths) < 1:
        raise InvalidInputError("GAP lengths must be positive")
    vol = math.prod(lengths)
    if vol > 1 << 14:
        raise InvalidInputError("GAP volume capped at 2^14")
    tot = np.full(1, a, dtype=np.int64)
    for s, n in zip(steps, lengths):
        tot = (tot[:, None] + np.arange(n, dtype=np.int64)[None, :] * s).reshape(-1)
    vals = np.unique(tot % N)
    return _support(N, vals), vals.size == vol


def union_of_elementary(a_n: int, etas, M: int, seed: int, alpha: float = 1.0, attempts: int = 100) -> SupportSet:
    """eta_i random elementary sets of size 2^i, i = 0..a_n, regenerated until
    a_n <= log2 |J| + alpha."""
    etas = [int(e) for e in etas]
    if len(etas) != a_n + 1:
        raise InvalidInputError("need one eta per size exponent 0..a_n")
    if a_n > M:
        raise InvalidInputError("a_n exceeds M")
    if not any(etas):
        raise InvalidInputError("empty union")
    for t in range(attempts):
        g = rng_from_seed(seed, 2, t)
        parts = [(np.arange(1 << i) + (g.integers(0, 1 << (M - i), size=1 << i) << i)) % (1 << M)
                 for i, eta in enumerate(etas) for _ in range(eta)]
        J = _support(1 << M, np.concatenate(parts))
        if a_n <= math.log2(len(J)) + alpha:
            return J
    raise ContractViolationError(f"could not realize a_n <= log2 k + {alpha} in {attempts} attempts")


def union_of_homogeneous(K: SupportSet, a_n: int, etas, seed: int, alpha: float = 1.0,
                         attempts: int = 100) -> SupportSet:
    """Union of subsets of a homogeneous K that vary its first i pivot bits."""
    cls = classify(K)
    if not cls.is_homogeneous:
        raise InvalidInputError("UoH base set must be homogeneous")
    lv = cls.pivots
    if a_n > len(lv):
        raise InvalidInputError("a_n exceeds the base pivot count")
    etas = [int(e) for e in etas]
    if len(etas) != a_n + 1:
        raise InvalidInputError("need one eta per size exponent 0..a_n")
    if not any(etas):
        raise InvalidInputError("empty union")
    arr = K.as_array()
    pat = np.zeros(arr.size, dtype=np.int64)
    for i, li in enumerate(lv):
        pat |= ((arr >> li) & 1) << i
    by_pat = np.empty(1 << len(lv), dtype=np.int64)
    by_pat[pat] = arr
    s = len(lv)
    for t in range(attempts):
        g = rng_from_seed(seed, 3, t)
        picks = []
        for i, eta in enumerate(etas):
            for _ in range(eta):
                fixed = (int(g.integers(0, 1 << (s - i))) << i) if s > i else 0
                picks.append(by_pat[fixed | np.arange(1 << i)])
        J = _support(K.N, np.concatenate(picks))
        if a_n <= math.log2(len(J)) + alpha:
            return J
    raise ContractViolationError(f"could not realize a_n <= log2 k + {alpha} in {attempts} attempts")


def bernoulli_subset(K: SupportSet, k: int, seed: int) -> SupportSet:
    """Each element of K kept with probability k/|K| (retried while empty)."""
    if not 1 <= k <= len(K):
        raise InvalidInputError("need 1 <= k <= |K|")
    arr = K.as_array()
    for t in range(100):
        keep = rng_from_seed(seed, 4, t).random(arr.size) < k / arr.size
        if keep.any():
            return _support(K.N, arr[keep])
    raise ContractViolationError("random subset repeatedly empty")


def bernoulli_subset_zn(M: int, k: int, seed: int) -> SupportSet:
    """Each j in Z_N kept with probability k/N (retried while empty)."""
    N = 1 << M
    if not 1 <= k <= N:
        raise InvalidInputError("need 1 <= k <= N")
    for t in range(100):
        hits = np.flatnonzero(rng_from_seed(seed, 4, t).random(N) < k / N)
        if hits.size:
            return _support(N, hits)
    raise ContractViolationError("random subset repeatedly empty")


def jstar(M: int) -> SupportSet:
    """{1, 2, 4, ..., 2^(M-1)}: a pivot at every level."""
    if M < 1:
        raise InvalidInputError("need M >= 1")
    return _support(1 << M, [1 << i for i in range(M)])


def doubling(J: SupportSet) -> int:
    """|J + J mod N| by enumeration (|J| <= 2^12)."""
    if len(J) > 1 << 12:
        raise InvalidInputError("doubling enumeration capped at |J| <= 2^12")
    a = J.as_array()
    return int(np.unique((a[:, None] + a[None, :]) % J.N).size)


@dataclass(frozen=True)
class Family:
    """One seeded family draw: the support and the policy metadata the SAS
    pivot selection uses (reference FamilySpec / FamilyInstance)."""
    kind: str
    support: SupportSet
    meta: dict


def build_family(kind: str, params: dict, seed: int = 0) -> Family:
    if kind not in KINDS:
        raise InvalidInputError(f"unknown family kind {kind!r}")
    p = dict(params)
    try:
        if kind == "elementary":
            return Family(kind, elementary(p["r"], p["M"], seed), {"policy": "uoe"})
        if kind == "homogeneous":
            return Family(kind, homogeneous(tuple(p["pivots"]), p["M"], seed), {"policy": "auto"})
        if kind in ("consecutive", "ap"):
            step = 1 if kind == "consecutive" else p["s"]
            return Family(kind, arithmetic(p["a"], step, p["k"], p["N"]), {"policy": "auto"})
        if kind == "gap":
            J, proper = generalized_ap(p["a"], p["steps"], p["lengths"], p["N"])
            return Family(kind, J, {"policy": "auto", "proper": proper})
        if kind == "uoe":
            return Family(kind, union_of_elementary(p["a_n"], p["etas"], p["M"], seed, p.get("alpha", 1.0)),
                          {"policy": "uoe"})
        if kind == "uoh":
            K = homogeneous(tuple(p["base_pivots"]), p["M"], seed + 1)
            J = union_of_homogeneous(K, p["a_n"], p["etas"], seed, p.get("alpha", 1.0))
            return Family(kind, J, {"policy": "uoh", "base_pivots": pivots(K)})
        if kind == "random_subset":
            if p.get("base", "zn") == "zn":
                return Family(kind, bernoulli_subset_zn(p["M"], p["k"], seed),
                              {"policy": "random_subset", "base_pivots": tuple(range(p["M"]))})
            K = homogeneous(tuple(p["base_pivots"]), p["M"], seed + 1)
            return Family(kind, bernoulli_subset(K, p["k"], seed),
                          {"policy": "random_subset", "base_pivots": pivots(K)})
        return Family(kind, jstar(p["M"]), {"policy": "auto"})
    except KeyError as e:
        raise InvalidInputError(f"family {kind!r} needs parameter {e}") from None
