"""Where the time goes in device SAS (config 3, reference policies)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402


B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
wl = W.make_workload(3, B)
sig = torch.empty((B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(sig, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
base = W.config_pivots(3)
lib = S._lib.load()
timers = {}
orig = {}
for name in ("sfft_hidft_shifts", "sfft_sas_decode", "sfft_plan_nodes", "sfft_prefix_weights", "sfft_pivoted_pattern"):
    fn = getattr(lib, name)
    orig[name] = fn

    def wrap(*a, _fn=fn, _n=name):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = _fn(*a)
        torch.cuda.synchronize()
        timers[_n] = timers.get(_n, 0.0) + time.perf_counter() - t0
        return rc
    setattr(lib, name, wrap)
for pol in ("auto", "random_subset"):
    S.sas_transform(sig, J, policy=pol, family_meta={"base_pivots": base})
    timers.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = S.sas_transform(sig, J, policy=pol, family_meta={"base_pivots": base})
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print(f"{pol}: total {tot * 1e3:.2f} ms  " + "  ".join(f"{k}={v * 1e3:.2f}ms" for k, v in timers.items()))
