"""Support sets and pivot analysis (reference congruence.py), device-backed.

`pivots(J)` and `classify(J)` run on the B200 (sfft_analyze: bit-reversed
bitmap rank + adjacent-pair levels, congruence.py:76-101) and are cached on
the immutable SupportSet, so a support is analysed once however many calls
reuse it (the reference re-derives it 2-3 times per call).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from .errors import ContractViolationError, InvalidInputError


def v2(x: int) -> int:
    """2-adic valuation of a nonzero integer (congruence.py:22-27)."""
    x = int(x)
    if x == 0:
        raise InvalidInputError("v2(0) is undefined")
    return (x & -x).bit_length() - 1


def _is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


class SupportSet:
    """A validated frequency support J, a nonempty subset of Z_N, N = 2^M.

    Same constructor, validation and messages as congruence.py:34-73; the
    indices are held as an int64 array (plus a lazily built tuple), with
    per-device copies and plan caches attached to the immutable object.
    """

    __slots__ = ("N", "_arr", "_tuple", "_dev", "_pivots", "_plans", "__weakref__")

    def __init__(self, N: int, indices):
        N = int(N)
        if not _is_power_of_two(N):
            raise InvalidInputError(f"N={N} is not a power of two")
        arr = np.asarray(indices, dtype=np.int64).reshape(-1)
        if arr.size == 0:
            raise InvalidInputError("support set is empty")
        if (arr < 0).any() or (arr >= N).any():
            raise InvalidInputError("support indices must lie in [0, N)")
        if arr.size > 1 and (np.diff(arr) <= 0).any():
            raise InvalidInputError("support indices must be strictly increasing")
        arr.setflags(write=False)
        object.__setattr__(self, "N", N)
        object.__setattr__(self, "_arr", arr)
        object.__setattr__(self, "_tuple", None)
        object.__setattr__(self, "_dev", {})
        object.__setattr__(self, "_pivots", None)
        object.__setattr__(self, "_plans", {})

    def __setattr__(self, name, value):
        raise AttributeError("SupportSet is immutable")

    @classmethod
    def make(cls, N: int, indices: Iterable[int]) -> "SupportSet":
        arr = np.asarray(list(indices) if not isinstance(indices, np.ndarray) else indices,
                         dtype=np.int64).reshape(-1)
        srt = np.sort(arr)
        if srt.size > 1 and (np.diff(srt) == 0).any():
            raise InvalidInputError("support indices must be distinct")
        return cls(N, srt)

    @property
    def indices(self) -> tuple[int, ...]:
        if self._tuple is None:
            object.__setattr__(self, "_tuple", tuple(int(j) for j in self._arr))
        return self._tuple

    @property
    def M(self) -> int:
        return self.N.bit_length() - 1

    def __len__(self) -> int:
        return int(self._arr.size)

    def __iter__(self):
        return iter(self.indices)

    def __contains__(self, j: int) -> bool:
        pos = int(np.searchsorted(self._arr, j))
        return pos < self._arr.size and int(self._arr[pos]) == int(j)

    def __eq__(self, other) -> bool:
        return (isinstance(other, SupportSet) and self.N == other.N
                and np.array_equal(self._arr, other._arr))

    def __hash__(self) -> int:
        return hash((self.N, self._arr.tobytes()))

    def __repr__(self) -> str:
        head = ", ".join(str(int(x)) for x in self._arr[:8])
        more = ", ..." if self._arr.size > 8 else ""
        return f"SupportSet(N={self.N}, k={len(self)}, indices=({head}{more}))"

    def as_array(self) -> np.ndarray:
        return self._arr.copy()

    def device_tensor(self, device):
        """int64 copy of the indices on `device`, cached."""
        import torch
        key = str(device)
        t = self._dev.get(key)
        if t is None:
            t = torch.from_numpy(self._arr.copy()).to(device, non_blocking=False)
            self._dev[key] = t
        return t


def as_support(J) -> SupportSet:
    """Accept our SupportSet or any object with .N and .indices (e.g. the
    reference's SupportSet)."""
    if isinstance(J, SupportSet):
        return J
    if type(J).__module__.startswith("torch"):
        raise InvalidInputError("expected a SupportSet, got a tensor")
    if hasattr(J, "N") and hasattr(J, "indices"):
        return SupportSet(J.N, np.asarray(J.indices, dtype=np.int64))
    raise InvalidInputError("expected a SupportSet")


def _mask_to_levels(mask: int) -> tuple[int, ...]:
    return tuple(i for i in range(64) if (mask >> i) & 1)


def pivots(J) -> tuple[int, ...]:
    """All levels l with some pair of J differing by an odd multiple of 2^l
    (congruence.py:76-101), computed on the device and cached on J."""
    J = as_support(J)
    if J._pivots is not None:
        return J._pivots
    if len(J) == 1:
        object.__setattr__(J, "_pivots", ())
        return ()
    if J.M > 31:
        raise InvalidInputError("device path supports N <= 2^31")
    dev = _lib.require_device()
    lib = _lib.load()
    dj = J.device_tensor(dev)
    mask = ctypes.c_uint64(0)
    homog = ctypes.c_int(0)
    _lib.check(lib.sfft_analyze(dj.data_ptr(), len(J), J.M, ctypes.byref(mask), ctypes.byref(homog),
                                _lib.stream_ptr(dev)))
    p = _mask_to_levels(mask.value)
    object.__setattr__(J, "_pivots", p)
    return p


@dataclass(frozen=True)
class Classification:
    kind: str  # "homogeneous" | "generic"
    pivots: tuple[int, ...]

    @property
    def is_homogeneous(self) -> bool:
        return self.kind == "homogeneous"


def classify(J) -> Classification:
    """Homogeneous iff |J| = 2^t with exactly t pivots (congruence.py:235-241)."""
    J = as_support(J)
    p = pivots(J)
    k = len(J)
    if _is_power_of_two(k) and len(p) == k.bit_length() - 1:
        return Classification("homogeneous", p)
    return Classification("generic", p)


def validate_pivot_vector(r: Sequence[int], M: int) -> tuple[int, ...]:
    """Strictly increasing levels in [0, M) (congruence.py:272-278)."""
    r = tuple(int(x) for x in r)
    if any(r[i] >= r[i + 1] for i in range(len(r) - 1)):
        raise InvalidInputError("pivot vector must be strictly increasing")
    if any(x < 0 or x >= M for x in r):
        raise InvalidInputError(f"pivots must lie in [0, {M})")
    return r


def is_part_homogeneous(J, r: Sequence[int]) -> bool:
    """Every pivot <= max(r) is listed in r (congruence.py:244-256)."""
    r = tuple(r)
    if not r:
        return True
    r_max, rset = max(r), set(r)
    return all(p in rset for p in pivots(J) if p <= r_max)


def assert_part_homogeneous(J, r: Sequence[int]) -> None:
    """congruence.py:259-269, same message."""
    r = tuple(r)
    if not r:
        return
    r_max, rset = max(r), set(r)
    for p in pivots(J):
        if p <= r_max and p not in rset:
            raise ContractViolationError(
                f"support is not {r}-part-homogeneous: pivot {p} <= {r_max} missing from r")


def height_of(level: int, r: Sequence[int]) -> int:
    """Number of pivots of r in [level, max(r)] (congruence.py:281-286)."""
    r = tuple(r)
    if not r:
        return 0
    return sum(1 for x in r if level <= x <= r[-1])


# ------------------------------------------------------ congruence tree ---

@dataclass(frozen=True)
class TreeNode:
    """A residue class mod 2^level meeting J (congruence.py:123-131)."""
    level: int
    residue: int
    members: tuple[int, ...]

    @property
    def weight(self) -> int:
        return len(self.members)


class CongruenceTree:
    """The mod-2^l refinement tree of J truncated at `depth` levels
    (congruence.py:134-214), built on the device by sfft_tree_build: per
    level, J sorted by rotr_M(j, l) is the node order (ascending residue,
    members ascending) and a node starts where neighbours differ in the low
    l bits.  The per-level arrays stay in numpy; TreeNode objects (tuples of
    members, as the reference stores them) are made on access."""

    def __init__(self, J, depth: int):
        J = as_support(J)
        if depth < 0 or depth > J.M:
            raise InvalidInputError(f"depth must be in [0, {J.M}]")
        self.support = J
        self.N = J.N
        self.M = J.M
        self.depth = int(depth)
        self._members, self._off, self._n = _tree_levels(J, 0, self.depth)
        self._levels = None

    # arrays ---------------------------------------------------------------
    def _residues(self, level: int) -> np.ndarray:
        n = int(self._n[level])
        return self._members[level][self._off[level][:n]] & ((1 << level) - 1)

    def node_weights(self, level: int) -> np.ndarray:
        """Weights of the nodes of `level` in ascending residue order."""
        self._check_level(level)
        n = int(self._n[level])
        return np.diff(self._off[level][:n + 1]).astype(np.int64)

    def _node_at(self, level: int, i: int) -> TreeNode:
        a, b = int(self._off[level][i]), int(self._off[level][i + 1])
        mem = self._members[level][a:b]
        return TreeNode(level, int(mem[0]) & ((1 << level) - 1), tuple(int(x) for x in mem))

    # reference interface --------------------------------------------------
    @property
    def levels(self) -> list:
        """[{residue: TreeNode}] per level, as the reference stores them."""
        if self._levels is None:
            self._levels = [{nd.residue: nd for nd in (self._node_at(l, i) for i in range(int(self._n[l])))}
                            for l in range(self.depth + 1)]
        return self._levels

    @property
    def root(self) -> TreeNode:
        return self._node_at(0, 0)

    def nodes_at_level(self, level: int) -> list:
        self._check_level(level)
        return [self._node_at(level, i) for i in range(int(self._n[level]))]

    def node(self, level: int, residue: int):
        self._check_level(level)
        res = self._residues(level)
        i = int(np.searchsorted(res, int(residue)))
        if i < res.size and int(res[i]) == int(residue):
            return self._node_at(level, i)
        return None

    def node_weight(self, level: int, residue: int) -> int:
        n = self.node(level, residue)
        return 0 if n is None else n.weight

    def induced_weight(self, level: int, residue: int, w) -> complex:
        """Sum of w over the node's members; 0 for absent nodes."""
        n = self.node(level, residue)
        if n is None:
            return 0j
        return complex(sum(w[j] for j in n.members))

    def children(self, node: TreeNode):
        """(left, right) children; left carries bit `node.level` set."""
        if node.level >= self.depth:
            raise InvalidInputError("node has no stored children (below tree depth)")
        right = self.node(node.level + 1, node.residue)
        left = self.node(node.level + 1, node.residue + (1 << node.level))
        return left, right

    def parent(self, node: TreeNode):
        if node.level == 0:
            return None
        return self.node(node.level - 1, node.residue % (1 << (node.level - 1)))

    def max_weight_at_level(self, level: int) -> int:
        return int(self.node_weights(level).max())

    def split_levels(self) -> tuple[int, ...]:
        """Levels (below depth) at which some stored node has two children."""
        return tuple(l for l in range(self.depth) if int(self._n[l + 1]) > int(self._n[l]))

    def _check_level(self, level: int) -> None:
        if level < 0 or level > self.depth:
            raise InvalidInputError(f"level {level} outside stored depth {self.depth}")


def _tree_levels(J: SupportSet, lo: int, hi: int):
    """(members (L, k) int64, node_off (L, k+1) int32, n_nodes (L,)) for levels lo..hi."""
    k = len(J)
    L = hi - lo + 1
    if J.M == 0:  # N = 1: the one-element tree
        return (np.zeros((L, 1), np.int64), np.tile(np.array([0, 1], np.int32), (L, 1)), np.ones(L, np.int32))
    dev = _lib.require_device()
    lib = _lib.load()
    dj = J.device_tensor(dev)
    members = np.empty((L, k), dtype=np.int64)
    off = np.empty((L, k + 1), dtype=np.int32)
    n = np.empty(L, dtype=np.int32)
    _lib.check(lib.sfft_tree_build(dj.data_ptr(), k, J.M, lo, hi, members.ctypes.data, off.ctypes.data,
                                   n.ctypes.data, _lib.stream_ptr(dev)))
    return members, off, n


def level_weights(J, level: int) -> np.ndarray:
    """Node weights of T(J) at one level, ascending residue (device)."""
    J = as_support(J)
    if level < 0 or level > J.M:
        raise InvalidInputError(f"depth must be in [0, {J.M}]")
    _, off, n = _tree_levels(J, level, level)
    return np.diff(off[0][:int(n[0]) + 1]).astype(np.int64)


def build_tree(J, depth: int, counter=None) -> CongruenceTree:
    """Construct T^depth(J) (congruence.py:217-222); counts |J| * depth bit
    operations like the reference."""
    J = as_support(J)
    tree = CongruenceTree(J, depth)
    if counter is not None:
        counter.count_bit_ops(len(J) * max(depth, 1))
    return tree
