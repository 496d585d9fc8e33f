"""SFFT_HOST_TRACE timeline of the config-5 public call on 64 page-locked host rows, plus Python-side costs."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2211_15299_b200 as S
from paper_2211_15299_b200 import workloads as W
wl = W.make_workload(5, B=64)
dev = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True); host.copy_(dev); del dev
J = S.SupportSet(wl.N, wl.support)
for i in range(4):
    t = time.perf_counter(); S.hidft_to_dft_batched(host, J); print("call ms", (time.perf_counter() - t) * 1e3, file=sys.stderr, flush=True)
from paper_2211_15299_b200.hidft import classify, get_plan, _lib
import paper_2211_15299_b200.hidft as H
for name, fn in [("pinned empty 32 MiB", lambda: torch.empty((wl.B, wl.k), dtype=torch.complex64, pin_memory=True)),
                 ("classify", lambda: classify(J)),
                 ("get_plan", lambda: get_plan(J, classify(J).pivots, 0, _lib.C64, torch.device("cuda", 0))),
                 ("device_tensor", lambda: J.device_tensor(torch.device("cuda", 0)))]:
    fn()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    print(name, "ms", (time.perf_counter() - t) * 100, file=sys.stderr, flush=True)
