"""SFFT_HOST_TRACE timeline of the config-2 public call on page-locked host rows."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
H = sys.modules["paper_2211_15299_b200.hidft"]  # the package re-exports the function hidft under that name
from paper_2211_15299_b200 import workloads as W  # noqa: E402

wl = W.make_workload(int(os.environ.get("CFG", "2")))
dev = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
host.copy_(dev)
del dev
J = S.SupportSet(wl.N, wl.support)
runs = [(c, t) for c in os.environ.get("CHUNKS", "0").split() for t in os.environ.get("THREADS", "0").split()]
for chunks, thr in [(int(c), int(t)) for c, t in runs]:
    H.HOST_CHUNK_ROWS = chunks
    H.HOST_GATHER_THREADS = thr
    per = []
    for i in range(8):
        t = time.perf_counter()
        S.hidft_to_dft_batched(host, J)
        per.append(time.perf_counter() - t)
    print(f"chunk rows {chunks} threads {thr}: call ms", " ".join(f"{x * 1e3:.3f}" for x in per), file=sys.stderr,
          flush=True)
