"""Config-5 end-to-end breakdown on host rows (B rows of the config, default 64):
whole public call, host gather alone (pattern order, as the split staging
reads it), and the raw page-locked copy rates for the same bytes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
H = sys.modules["paper_2211_15299_b200.hidft"]  # the package re-exports the function hidft under that name
from paper_2211_15299_b200 import _lib, workloads as W  # noqa: E402
from paper_2211_15299_b200.hidft import get_plan  # noqa: E402

B = int(os.environ.get("B", "64"))
wl = W.make_workload(5, B=B)
dev = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
t = time.perf_counter()
host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
print(f"pin_memory {host.numel() * 8 / 2**30:.0f} GiB: {time.perf_counter() - t:.1f} s", flush=True)
host.copy_(dev)
del dev
torch.cuda.empty_cache()
J = S.SupportSet(wl.N, wl.support)


def timeit(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


for chunks in (0, 8, 16, 32):
    H.HOST_CHUNK_ROWS = chunks
    dt = timeit(lambda: S.hidft_to_dft_batched(host, J))
    print(f"public call, chunk rows {chunks or 'default'}: {dt * 1e3:.2f} ms  {wl.B * wl.k / dt:.3e} coeffs/s", flush=True)
H.HOST_CHUNK_ROWS = 0
plan = get_plan(J, S.pivots(J), 0, _lib.C64, torch.device("cuda", 0))
offs = plan.tables()["offsets"]
pat = np.sort(offs).astype(np.int64)
stage = torch.empty((wl.B, plan.A), dtype=torch.complex64, pin_memory=True)
lib = _lib.load()
for thr in (0, 8):
    dt = timeit(lambda: lib.sfft_host_gather(host.data_ptr(), wl.B, wl.N, 8, pat.ctypes.data, plan.A,
                                             stage.data_ptr(), thr))
    print(f"host gather only (pattern order), threads {thr or 'default'}: {dt * 1e3:.2f} ms "
          f"({stage.numel() * 8 / dt / 1e9:.1f} GB/s)", flush=True)
dstage = torch.empty((wl.B, plan.A), dtype=torch.complex64, device="cuda")
h2d = timeit(lambda: dstage.copy_(stage, non_blocking=True))
d2h = timeit(lambda: stage.copy_(dstage, non_blocking=True))
nb = stage.numel() * 8
print(f"H2D {nb / 2**20:.0f} MiB: {h2d * 1e3:.2f} ms ({nb / h2d / 1e9:.1f} GB/s); D2H: {d2h * 1e3:.2f} ms "
      f"({nb / d2h / 1e9:.1f} GB/s)")
