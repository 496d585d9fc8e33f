"""Pure-write, pure-read and copy bandwidth of the box (torch kernels, CUDA events): bounds for the split passes."""
import torch
n = 1 << 28  # 1 GiB of fp32
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
def t(f, reps=10):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best * 1e-3
GB = n * 4 / 1e9
print("write-only (fill_): %.0f GB/s" % (GB / t(lambda: a.fill_(1.0))))
print("write-only (zero_/memset): %.0f GB/s" % (GB / t(lambda: a.zero_())))
print("read-only (sum): %.0f GB/s" % (GB / t(lambda: a.sum())))
print("copy: %.0f GB/s total" % (2 * GB / t(lambda: b.copy_(a))))
for mb in (16, 32, 64, 128):
    m = mb << 18
    print("write-only %d MiB (fill_): %.0f GB/s" % (mb, m * 4 / 1e9 / t(lambda: a[:m].fill_(1.0), 30)))
