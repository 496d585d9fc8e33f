"""Python-side cost of the public host-rows call (config 1, tiny batch): cProfile of 300 calls."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402

wl = W.make_workload(1)
dev = torch.empty((wl.B, wl.N), dtype=torch.complex128, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
host.copy_(dev)
J = S.SupportSet(wl.N, wl.support)
for _ in range(20):
    S.hidft_to_dft_batched(host, J)
t = time.perf_counter()
for _ in range(300):
    S.hidft_to_dft_batched(host, J)
print("per call us", (time.perf_counter() - t) / 300 * 1e6)
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    S.hidft_to_dft_batched(host, J)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
