"""Small run of every kernel family, for compute-sanitizer (one tool per call)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2211_15299_b200 as S  # noqa: E402
import structfft_oracle as O  # noqa: E402

rng = np.random.default_rng(1)
# plan kernel (shared support), c64 and c128, with shift and height
J = O.gen_homogeneous((0, 2, 3, 5, 7, 9), 14, 3)
Js = S.SupportSet(1 << 14, J)
f = torch.randn(4, 1 << 14, dtype=torch.complex64, device="cuda")
S.hidft(f, Js, S.pivots(Js), shift=77)
S.hidft(f.to(torch.complex128), Js, S.pivots(Js), height=2)
S.hidft_to_dft_batched(f, Js)
# fused per-signal
sup = np.stack([O.gen_homogeneous(sorted(rng.choice(14, size=6, replace=False).tolist()), 14, int(rng.integers(1 << 30))) for _ in range(4)])
S.hidft_to_dft_batched(f, torch.from_numpy(sup).cuda())
# split transform (s = 15 and 16, c64; s = 14 c128), device rows and host rows
J2 = O.gen_homogeneous(sorted(rng.choice(20, size=15, replace=False).tolist()), 20, 5)
f2 = torch.randn(2, 1 << 20, dtype=torch.complex64, device="cuda")
S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J2))
S.hidft_to_dft_batched(f2.cpu(), S.SupportSet(1 << 20, J2))
J3 = np.arange(1 << 16, dtype=np.int64) * 4 + 1
S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J3))
J4 = np.arange(1 << 14, dtype=np.int64) * 8 + 3
S.hidft(f2[0].to(torch.complex128), S.SupportSet(1 << 20, J4), S.pivots(S.SupportSet(1 << 20, J4)), shift=9)
# host paths: shared support, per-signal supports, SAS staging
S.hidft_to_dft_batched(f.cpu(), Js)
S.hidft_to_dft_batched(f.cpu(), torch.from_numpy(sup))
# SAS mu* > 1 with escalation, band-limited source
H = O.gen_homogeneous((0, 2, 3, 5, 7, 9, 10), 14, 4)
Jsub = np.sort(H[rng.choice(H.size, size=40, replace=False)])
Jb = S.SupportSet(1 << 14, Jsub)
c = rng.normal(size=40) + 1j * rng.normal(size=40)
S.sas_transform(S.BandlimitedSignal(Jb, c), Jb, policy="random_subset", family_meta={"base_pivots": (0, 2, 3, 5, 7, 9, 10)})
fb = S.BandlimitedSignal(Jb, c).synthesize()
fb = fb.cpu().numpy() if hasattr(fb, "cpu") else np.asarray(fb)
S.sas_transform(np.stack([fb, fb]), Jb, policy="random_subset", family_meta={"base_pivots": (0, 2, 3, 5, 7, 9, 10)})
S.sas_transform(torch.from_numpy(np.stack([fb, fb])).cuda(), Jb, policy="random_subset",
                family_meta={"base_pivots": (0, 2, 3, 5, 7, 9, 10)})
# TMA head + final (s = 16 c64 with pivots M-2, M-1: two row chunks via a small scratch budget is
# not settable here, so three rows), and the three-pass fallback for a shifted call
J6 = O.gen_homogeneous(sorted(rng.choice(18, size=14, replace=False).tolist()) + [18, 19], 20, 7)
S.hidft_to_dft_batched(torch.randn(3, 1 << 20, dtype=torch.complex64, device="cuda"), S.SupportSet(1 << 20, J6))
S.hidft(f2, S.SupportSet(1 << 20, J6), S.pivots(S.SupportSet(1 << 20, J6)), shift=5)
# back-to-back calls in a PDL chain scope, 2^14-slot plan kernel (32 slots per thread)
with S.stream_chain():
    for _ in range(3):
        S.hidft_to_dft_batched(f, Js)
        S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J3))
        S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J6))
J5 = O.gen_homogeneous(sorted(rng.choice(20, size=14, replace=False).tolist()), 20, 6)
S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J5))
S.hidft_to_dft_batched(f2, S.SupportSet(1 << 20, J5))
torch.cuda.synchronize()
print("sanitize case ok")
