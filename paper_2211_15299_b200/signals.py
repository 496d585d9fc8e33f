"""Band-limited signals synthesised on the device (reference core.py:129-177).

`BandlimitedSignal(J, coeffs)` keeps the reference interface (coeff,
coeff_map, sample, sample_block, synthesize); samples are evaluated by the
`sfft_synthesize` kernel in float64 with the exponent reduced exactly in
integer arithmetic, so a Hi-DFT over a BandlimitedSignal source runs fully on
the GPU (hidft() synthesises only the 2^s samples it needs, in slot order).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .congruence import as_support
from .errors import InvalidInputError


class BandlimitedSignal:
    def __init__(self, support, coeffs):
        self.support = as_support(support)
        self.N = self.support.N
        c = np.asarray(coeffs, dtype=np.complex128)
        if c.shape != (len(self.support),):
            raise InvalidInputError(f"need exactly {len(self.support)} coefficients, got shape {c.shape}")
        if not np.all(np.isfinite(c)):
            raise InvalidInputError("coefficients contain NaN or Inf")
        self.coeffs = c
        self._l = self.support.as_array()
        self._dev = {}

    @classmethod
    def from_reference(cls, sig) -> "BandlimitedSignal":
        """Wrap the reference's BandlimitedSignal (anything with .support/.coeffs)."""
        return sig if isinstance(sig, cls) else cls(as_support(sig.support), sig.coeffs)

    def coeff(self, j: int) -> complex:
        pos = int(np.searchsorted(self._l, j))
        if pos >= len(self._l) or self._l[pos] != j:
            raise InvalidInputError(f"index {j} not in support")
        return complex(self.coeffs[pos])

    def coeff_map(self) -> dict[int, complex]:
        return {int(l): complex(c) for l, c in zip(self._l, self.coeffs)}

    def _device(self, device):
        import torch
        key = str(device)
        if key not in self._dev:
            self._dev[key] = (self.support.device_tensor(device),
                              torch.from_numpy(self.coeffs.copy()).to(device))
        return self._dev[key]

    def sample_block_tensor(self, locations):
        """Samples at `locations` (int64 tensor on a CUDA device) as a complex128 tensor."""
        import torch
        loc = locations.to(torch.int64).contiguous()
        J, c = self._device(loc.device)
        out = torch.empty(loc.numel(), dtype=torch.complex128, device=loc.device)
        _lib.check(_lib.load().sfft_synthesize(J.data_ptr(), c.data_ptr(), len(self.support), self.support.M,
                                               loc.data_ptr(), loc.numel(), out.data_ptr(),
                                               _lib.stream_ptr(loc.device)))
        return out.view(loc.shape)

    def sample_block(self, locations) -> np.ndarray:
        import torch
        dev = _lib.require_device()
        loc = torch.as_tensor(np.asarray(locations, dtype=np.int64) % self.N, device=dev)
        return self.sample_block_tensor(loc).cpu().numpy()

    def sample(self, i: int) -> complex:
        if i < 0 or i >= self.N:
            raise InvalidInputError(f"sample index {i} out of range [0, {self.N})")
        return complex(self.sample_block(np.asarray([i]))[0])

    def synthesize(self) -> np.ndarray:
        return self.sample_block(np.arange(self.N))
