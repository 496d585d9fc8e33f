"""Per-phase cycle breakdown of the cluster kernel (debug timing build)."""
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
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
wl = W.make_workload(cfg, B)
cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
sig = torch.empty((B, wl.N), dtype=cdt, device="cuda")
W.synthesize_into(sig, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
for _ in range(3):
    out = S.hidft_to_dft_batched(sig, J)
torch.cuda.synchronize()
lib = _lib.load()
lib.sfft_debug_stamps.argtypes = [ctypes.c_void_p, ctypes.c_int]
plan = S.get_plan(J, S.pivots(J), 0, 0 if cdt == torch.complex64 else 1, torch.device("cuda", 0))
C = {16: 16, 15: 8, 17: 16}.get(plan.s, 16) if cdt == torch.complex64 else {14: 4, 15: 8, 16: 16}[plan.s]
nb = min(B * C, 148 * 4)
st = np.zeros((nb, 8), np.uint64)
_lib.check(lib.sfft_debug_stamps(st.ctypes.data, nb))
st = st.astype(np.int64)
st = st[st[:, 0] != 0]
rel = st - st[:, :1]
names = ["gather+stage", "push R1 + wait", "local stages", "push R2 + wait", "last stages+store"]
d = np.diff(st[:, :6], axis=1)
print(f"cfg{cfg} B={B} s={plan.s} C={C}: per-CTA cycles by phase (median / p90)")
for i, n in enumerate(names):
    print(f"  {n:18s} {np.median(d[:, i]):9.0f} {np.percentile(d[:, i], 90):9.0f}")
print(f"  {'total (last signal)':18s} {np.median(rel[:, 5]):9.0f}")
span = st[:, 5].max() - st[:, 0].min()
print(f"kernel span (cycles, SM clocks differ per SM -> indicative) {span}")

