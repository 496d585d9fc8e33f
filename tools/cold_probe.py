import time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2211_15299_b200 as S
from paper_2211_15299_b200 import workloads as W
sup = W.config_supports_batch(4, 4)
J = torch.from_numpy(sup).cuda()
row = torch.zeros((1, 1 << 20), dtype=torch.complex64, device="cuda")
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter(); S.hidft_to_dft_batched(row, J[:1], check=False); torch.cuda.synchronize(); print("fused call", i, (time.perf_counter()-t0)*1e3, "ms")
big = torch.empty((64 << 30) // 8, dtype=torch.complex64, device="cuda"); del big; torch.cuda.empty_cache()
J2 = torch.from_numpy(W.config_supports_batch(4, 2)[1:]).cuda()
t0 = time.perf_counter(); S.hidft_to_dft_batched(row, J2, check=False); torch.cuda.synchronize(); print("after 64 GiB alloc/free", (time.perf_counter()-t0)*1e3, "ms")
sup6, M = W.config_support(6)
from paper_2211_15299_b200.hidft import get_plan
for i in range(2):
    Js = S.SupportSet(1 << M, sup6)
    t0 = time.perf_counter(); get_plan(Js, S.pivots(Js), 0, 1, torch.device("cuda", 0)); torch.cuda.synchronize(); print("c128 plan", i, (time.perf_counter()-t0)*1e3, "ms")
