import ctypes, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2211_15299_b200 as S
from paper_2211_15299_b200 import workloads as W, _lib
from paper_2211_15299_b200.hidft import get_plan
wl = W.make_workload(5, B=2)
J = S.SupportSet(wl.N, wl.support)
plan = get_plan(J, S.pivots(J), 0, _lib.C64, torch.device("cuda", 0))
print("plan A", plan.A)
