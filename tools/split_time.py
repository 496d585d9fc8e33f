"""Time the config-5 transform (split path) with CUDA events, no parity gate:
for ablations through SFFT_SPLIT_DEBUG (bit 1 skip stores, bit 2 skip the
butterfly, bit 3 coalesced stores) and SFFT_SPLIT_SCRATCH_MB."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = W.make_workload(cfg)
cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
sig = torch.empty((wl.B, wl.N), dtype=cdt, device="cuda")
W.synthesize_into(sig, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
out = torch.empty((wl.B, wl.k), dtype=cdt, device="cuda")
for _ in range(3):
    S.hidft_to_dft_batched(sig, J, out=out, check=False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(10):
    S.hidft_to_dft_batched(sig, J, out=out, check=False)
e1.record()
torch.cuda.synchronize()
print(f"cfg{cfg} debug={os.environ.get('SFFT_SPLIT_DEBUG', '0')} scratch={os.environ.get('SFFT_SPLIT_SCRATCH_MB', 'default')}: "
      f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us per batch")
