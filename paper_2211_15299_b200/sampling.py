"""Pivoted multi-coset sample sets I_r (reference sampling.py:28-71), device-built."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .congruence import SupportSet, validate_pivot_vector


@dataclass(frozen=True)
class SamplingPattern:
    N: int
    pivots: tuple[int, ...]
    samples: tuple[int, ...]

    @property
    def M(self) -> int:
        return self.N.bit_length() - 1

    def __len__(self) -> int:
        return len(self.samples)

    def as_array(self) -> np.ndarray:
        return np.asarray(self.samples, dtype=np.int64)

    def as_support(self) -> SupportSet:
        return SupportSet.make(self.N, self.samples)


def pivoted_pattern_tensor(r: Sequence[int], M: int, device=None):
    """I_r ascending as a device int64 tensor (sampling.py:62-71)."""
    import torch
    rt = validate_pivot_vector(r, M)
    dev = device or _lib.require_device()
    out = torch.empty(1 << len(rt), dtype=torch.int64, device=dev)
    rr = np.asarray(rt if rt else [0], dtype=np.int32)
    _lib.check(_lib.load().sfft_pivoted_pattern(rr.ctypes.data, len(rt), M, out.data_ptr(),
                                                _lib.stream_ptr(dev)))
    return out


def pivoted_pattern(r: Sequence[int], M: int) -> SamplingPattern:
    """I_r = {sum_k b_k 2^(M-1-r_k)} sorted ascending (sampling.py:62-71)."""
    rt = validate_pivot_vector(r, M)
    t = pivoted_pattern_tensor(rt, M)
    return SamplingPattern(1 << M, rt, tuple(int(x) for x in t.cpu().numpy()))
