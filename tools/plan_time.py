"""Cold-call plan build time (fresh SupportSet -> device plan, synchronised) per config."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402
from paper_2211_15299_b200.hidft import get_plan  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.init()
for cfg in (1, 2, 3, 5, 6):
    sup, M = W.config_support(cfg)
    code = 0 if W.CONFIGS[cfg]["dtype"] == "complex64" else 1
    times = []
    for rep in range(4):
        J = S.SupportSet(1 << M, sup)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        get_plan(J, S.pivots(J), 0, code, dev)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    print(f"cfg {cfg}: plan ms first {times[0]:.3f} then {min(times[1:]):.3f}")
