"""Device time of hidft_to_dft_batched on config-5/6-shaped rows (no parity
gate: for probe variants of the library selected with SFFT_LIB)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402

cfg = int(os.environ.get("CFG", "5"))
wl = W.make_workload(cfg)
B = int(os.environ.get("B", wl.B))
dt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
sig = torch.randn((B, wl.N), dtype=dt, device="cuda")
J = S.SupportSet(wl.N, wl.support)
for _ in range(3):
    S.hidft_to_dft_batched(sig, J)
torch.cuda.synchronize()
st = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
n = 20
ev[0].record(st)
for _ in range(n):
    S.hidft_to_dft_batched(sig, J)
ev[1].record(st)
torch.cuda.synchronize()
print(f"cfg {cfg} B {B} lib {os.environ.get('SFFT_LIB', 'default')}: {ev[0].elapsed_time(ev[1]) / n * 1e3:.1f} us per call")
