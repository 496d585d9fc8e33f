"""Timing of device shift-and-sample on config 3 under the reference's policies."""
import os
import sys
import time

import numpy as np
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
for pol in ("auto", "random_subset"):
    for _ in range(2):
        res = S.sas_transform(sig, J, policy=pol, family_meta={"base_pivots": base})
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        res = S.sas_transform(sig, J, policy=pol, family_meta={"base_pivots": base})
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    got = res.coeffs.cpu().numpy()
    err = np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)
    print(f"cfg3 B={B} policy={pol:13s} s={len(res.plan.pivots)} mu*={res.plan.mu_star} "
          f"escalated={res.report.escalated_nodes} fallbacks={res.report.dense_fallbacks}: "
          f"{dt * 1e3:8.2f} ms/batch  {B * wl.k / dt:.3e} coeffs/s  max rel L2 vs planted {err.max():.2e}")
