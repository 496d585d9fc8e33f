"""Kernel-level timing of the Hi-DFT variants on one config (dev tool).

Times each variant over rotating input sets (cold L2), CUDA events on the
launching stream; prints one line per variant.
"""
import argparse
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import _lib, workloads as W  # noqa: E402


def timeit(fn, R, steps=200, warm=20):
    for i in range(warm):
        fn(i % R)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(steps):
        fn(i % R)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--sets", type=int, default=8)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    spec = W.CONFIGS[a.config]
    B = a.batch or spec["B"]
    wl = W.make_workload(a.config, B)
    cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
    esz = 8 if cdt == torch.complex64 else 16
    R = a.sets
    free = torch.cuda.mem_get_info()[0]
    R = max(1, min(R, int(free * 0.8 // (B * wl.N * esz))))
    sets = [torch.empty((B, wl.N), dtype=cdt, device="cuda") for _ in range(R)]
    W.synthesize_into(sets[0], wl.support, wl.coeffs)
    for s in sets[1:]:
        s.copy_(sets[0])
    out = torch.empty((B, wl.k), dtype=cdt, device="cuda")
    lib = _lib.load()
    stream = _lib.stream_ptr()
    res = {}
    if wl.support.ndim == 1:
        J = S.SupportSet(wl.N, wl.support)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        jt = J.device_tensor(torch.device("cuda"))
        code = _lib.C64 if esz == 8 else _lib.C128

        def fused(i):
            _lib.check(lib.sfft_hidft_to_dft_fused(jt.data_ptr(), wl.k, 1, wl.M, sets[i].data_ptr(), B, wl.N,
                                                   code, out.data_ptr(), wl.k, st.data_ptr(), stream))
        r = S.pivots(J)
        plan = S.get_plan(J, r, 0, code, torch.device("cuda", 0))
        kind = _lib.OUT_DFT if S.classify(J).is_homogeneous else _lib.OUT_SAS

        def planned(i):
            _lib.check(lib.sfft_hidft(plan.handle, sets[i].data_ptr(), B, wl.N, 0, kind, out.data_ptr(),
                                      wl.k, None, 0, stream))
        if S.classify(J).is_homogeneous:
            try:
                res["fused_shared"] = timeit(fused, R, a.steps)
            except Exception as e:
                print("fused:", e)
        try:
            res["plan_kernel"] = timeit(planned, R, a.steps)
            res["plan_kernel_hot_L2"] = timeit(planned, 1, a.steps)
        except Exception as e:
            print("plan:", e)
    else:
        jt = torch.from_numpy(wl.support).cuda()
        st = torch.zeros(B, dtype=torch.int32, device="cuda")

        def fused_ps(i):
            _lib.check(lib.sfft_hidft_to_dft_fused(jt.data_ptr(), wl.k, B, wl.M, sets[i].data_ptr(), B, wl.N,
                                                   _lib.C64, out.data_ptr(), wl.k, st.data_ptr(), stream))
        res["fused_per_signal"] = timeit(fused_ps, R, a.steps)
    for k, v in res.items():
        print(f"cfg{a.config} B={B} {k:22s} {v:9.2f} us/step  {B * wl.k / v * 1e6:.3e} coeffs/s")


if __name__ == "__main__":
    main()
