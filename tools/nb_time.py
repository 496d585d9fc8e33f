"""Device time of hidft_to_dft_interleaved on config-2-shaped data stored (N, B): a CUDA graph of 32 calls over
32 shifts (disjoint sample rows, as bench.py's layouts.interleaved) inside a stream_chain scope."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402

wl = W.make_workload(2)
rows = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(rows, wl.support, wl.coeffs)
nb = rows.T.contiguous()
del rows
J = S.SupportSet(wl.N, wl.support)
out = torch.empty((wl.B, wl.k), dtype=torch.complex64, device="cuda")
for i in range(4):
    S.hidft_to_dft_interleaved(nb, J, out=out, shift=i)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    with S.stream_chain():
        for i in range(32):
            S.hidft_to_dft_interleaved(nb, J, out=out, shift=i)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10):
    g.replay()
ev[1].record()
torch.cuda.synchronize()
print(f"interleaved cfg2 lib {os.environ.get('SFFT_LIB', 'default')}: {ev[0].elapsed_time(ev[1]) / 320 * 1e3:.2f} us per call (32-call graphs)")
