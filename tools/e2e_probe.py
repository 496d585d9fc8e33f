"""End-to-end (host-resident signals) timing of hidft_to_dft_batched vs pipeline knobs."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
H = sys.modules["paper_2211_15299_b200.hidft"]  # the package re-exports the function hidft under that name
from paper_2211_15299_b200 import workloads as W  # noqa: E402

wl = W.make_workload(2)
dev = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
host.copy_(dev)
J = S.SupportSet(wl.N, wl.support)
for thr in (0,):
    for chunks in (0,):
        H.HOST_GATHER_THREADS, H.HOST_CHUNK_ROWS = thr, chunks
        for _ in range(3):
            S.hidft_to_dft_batched(host, J)
        t0 = time.perf_counter()
        for _ in range(10):
            S.hidft_to_dft_batched(host, J)
        dt = (time.perf_counter() - t0) / 10
        print(f"gpu fraction {os.environ.get('SFFT_HOST_GPU_FRACTION', 'default')} threads {thr:2d} chunks {chunks:2d}: "
              f"{dt * 1e3:6.3f} ms/step  {wl.B * wl.k / dt:.3e} coeffs/s")

if os.environ.get("E2E_PROBE_FULL"):  # host gather alone, and the raw copy rates
    # host gather alone (no device work), same rows and locations
    import ctypes  # noqa: E402
    import numpy as np  # noqa: E402
    from paper_2211_15299_b200 import _lib  # noqa: E402
    from paper_2211_15299_b200.hidft import get_plan  # noqa: E402

    plan = get_plan(J, S.pivots(J), 0, _lib.C64, torch.device("cuda", 0))
    loc = np.ascontiguousarray(plan.tables()["offsets"], dtype=np.int64)
    stage = torch.empty((wl.B, plan.A), dtype=torch.complex64, pin_memory=True)
    lib = _lib.load()
    for thr in (0, 4, 8, 12, 15):
        for _ in range(2):
            lib.sfft_host_gather(host.data_ptr(), wl.B, wl.N, 8, loc.ctypes.data, plan.A, stage.data_ptr(), thr)
        t0 = time.perf_counter()
        for _ in range(10):
            lib.sfft_host_gather(host.data_ptr(), wl.B, wl.N, 8, loc.ctypes.data, plan.A, stage.data_ptr(), thr)
        dt = (time.perf_counter() - t0) / 10
        print(f"host gather only, threads {thr:2d}: {dt * 1e3:6.3f} ms")
    dstage = torch.empty((wl.B, plan.A), dtype=torch.complex64, device="cuda")
    for _ in range(3):
        dstage.copy_(stage, non_blocking=True)
        stage.copy_(dstage, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        dstage.copy_(stage, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(10):
        stage.copy_(dstage, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    nb = stage.numel() * 8
    print(f"H2D 8 MiB: {(t1 - t0) / 10 * 1e3:.3f} ms ({nb / ((t1 - t0) / 10) / 1e9:.1f} GB/s); "
          f"D2H: {(t2 - t1) / 10 * 1e3:.3f} ms ({nb / ((t2 - t1) / 10) / 1e9:.1f} GB/s)")
