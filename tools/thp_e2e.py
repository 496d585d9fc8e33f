"""e2e config-2 call on host rows in 4 KiB pages (torch pin_memory) vs
transparent huge pages (mmap + MADV_HUGEPAGE), pageable and page-locked."""
import ctypes
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_15299_b200 as S  # noqa: E402
from paper_2211_15299_b200 import workloads as W  # noqa: E402

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_HUGEPAGE = 14


def thp_array(shape, dtype):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    m = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    off = (-base) % (2 << 20)
    rc = libc.madvise(base + off, nbytes, MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.uint8, count=nbytes, offset=off).view(dtype).reshape(shape)
    return a, m, rc


def anon_huge_kb(addr):
    cur = None
    for line in open("/proc/self/smaps"):
        if "-" in line.split()[0] and len(line.split()[0].split("-")) == 2 and not line.startswith(("Anon", "Rss")):
            try:
                lo, hi = (int(x, 16) for x in line.split()[0].split("-"))
                cur = lo <= addr < hi
            except ValueError:
                pass
        elif cur and line.startswith("AnonHugePages"):
            return int(line.split()[1])
    return -1


wl = W.make_workload(2)
dev = torch.empty((wl.B, wl.N), dtype=torch.complex64, device="cuda")
W.synthesize_into(dev, wl.support, wl.coeffs)
J = S.SupportSet(wl.N, wl.support)
want = S.hidft_to_dft_batched(dev, J).cpu().numpy()


def timeit(name, host):
    for _ in range(3):
        out = S.hidft_to_dft_batched(host, J)
    got = np.asarray(out.cpu() if hasattr(out, "cpu") else out)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    per = []
    for _ in range(20):
        t = time.perf_counter()
        S.hidft_to_dft_batched(host, J)
        per.append(time.perf_counter() - t)
    per.sort()
    print(f"{name:40s} median {per[10] * 1e3:.3f} ms  min {per[0] * 1e3:.3f} ms  "
          f"{wl.B * wl.k / per[10]:.3e} coeffs/s  err {err:.1e}", flush=True)


pinned = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
pinned.copy_(dev)
timeit("torch pin_memory (cudaHostAlloc)", pinned)
print("pin_memory AnonHugePages kB:", anon_huge_kb(pinned.data_ptr()))
del pinned

a, m, rc = thp_array(tuple(dev.shape), np.complex64)
a[...] = dev.cpu().numpy()
print("madvise rc", rc, "AnonHugePages kB:", anon_huge_kb(a.ctypes.data))
timeit("THP numpy (pageable)", a)
t = torch.from_numpy(a)
timeit("THP torch CPU tensor (pageable)", t)
cr = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, a.nbytes, 0)
print("cudaHostRegister", cr)
timeit("THP + cudaHostRegister", t)
print("after register AnonHugePages kB:", anon_huge_kb(a.ctypes.data))
