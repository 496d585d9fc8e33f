import os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_2211_15299_b200 as S
from paper_2211_15299_b200 import workloads as W
B = 512
wl = W.make_workload(3, B)
sig = torch.empty((B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(sig, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
base = W.config_pivots(3)
for pol in ("auto", "random_subset"):
    for _ in range(2):
        res = S.sas_transform(sig, J, policy=pol, family_meta={"base_pivots": base})
torch.cuda.synchronize()
