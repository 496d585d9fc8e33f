"""Per-phase cycle totals of the fused split kernel (timing build,
tools/build_timing.sh): accumulated per CTA over its rows."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["SFFT_LIB"] = os.path.join(ROOT, "tools", "libsfft_b200_timing.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import _lib, workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = W.make_workload(cfg)
cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
sig = torch.empty((wl.B, wl.N), dtype=cdt, device="cuda")
W.synthesize_into(sig, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
out = torch.empty((wl.B, wl.k), dtype=cdt, device="cuda")
for _ in range(3):
    S.hidft_to_dft_batched(sig, J, out=out, check=False)
lib = _lib.load()
lib.sfft_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.sfft_debug_reset.argtypes = [ctypes.c_int]
nb = 148 * 4
_lib.check(lib.sfft_debug_reset(nb))
S.hidft_to_dft_batched(sig, J, out=out, check=False)
st = np.zeros((nb, 8), np.uint64)
_lib.check(lib.sfft_debug_stamps(st.ctypes.data, nb))
st = st.astype(np.float64)
live = st[:, :7].sum(1) > 0
st = st[live]
names = ["front issue", "wait front(i)", "stage block", "butterfly", "stores", "wait samples", "front finish"]
tot = st[:, :7].sum(1)
print(f"cfg{cfg}: {live.sum()} CTAs; per-CTA total cycles median {np.median(tot):.0f}")
for i, n in enumerate(names):
    print(f"  {n:14s} median {np.median(st[:, i]):10.0f}  ({np.median(st[:, i]) / np.median(tot) * 100:5.1f}%)")
