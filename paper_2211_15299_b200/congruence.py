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
