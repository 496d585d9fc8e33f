// Host memory rates on the GPU box: sequential read bandwidth vs isolated
// 8 B reads (one per 256 B, the config-2 minimum sample gap) vs one read per
// 128 B line pair, 16 threads over an 8 GiB buffer.  Tells whether the
// host gather is bound by DRAM bandwidth (buddy-line prefetch doubles the
// lines moved) or by memory-level parallelism.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <omp.h>
#include <vector>

int main() {
  const size_t n = (size_t)1 << 30;  // 8 GiB of uint64
  uint64_t* a = (uint64_t*)aligned_alloc(4096, n * 8);
#pragma omp parallel for
  for (size_t i = 0; i < n; ++i) a[i] = i;
  auto timeit = [&](const char* name, size_t stride, size_t count, double bytes_per) {
    double best = 1e30;
    uint64_t sink = 0;
    for (int rep = 0; rep < 5; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      uint64_t s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
      for (size_t i = 0; i < count; ++i) s += a[(i * stride) & (n - 1)];
      auto t1 = std::chrono::steady_clock::now();
      sink += s;
      best = std::min(best, std::chrono::duration<double>(t1 - t0).count());
    }
    printf("%-44s %8.3f ms  %7.1f GB/s of %5.0f B units  %.3e reads/s  (%llu)\n", name, best * 1e3,
           count * bytes_per / best / 1e9, bytes_per, count / best, (unsigned long long)(sink & 1));
  };
  printf("threads %d\n", omp_get_max_threads());
  timeit("sequential read (8 GiB)", 1, n, 8);
  // a large odd stride in elements scatters the reads over the buffer
  timeit("isolated 8 B reads, 1M, stride 32+ el (256 B)", 32 * 4099, 1 << 20, 64);
  timeit("isolated 8 B reads, 4M", 32 * 4099, 1 << 22, 64);
  timeit("reads 256 B apart, sequential order, 4M", 32, 1 << 22, 64);
  timeit("reads 128 B apart, sequential order, 4M", 16, 1 << 22, 64);
  timeit("reads 64 B apart, sequential order, 4M", 8, 1 << 22, 64);
  return 0;
}
