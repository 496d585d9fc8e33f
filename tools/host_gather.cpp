// Host-side gather rate: 1024 rows x 1024 isolated 8 B samples from an 8 GiB
// buffer into a contiguous 8 MiB staging buffer, OpenMP over rows.
// Variants: plain loop vs software prefetch D samples ahead (flattened over
// rows), for several thread counts.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <omp.h>
#include <sys/mman.h>
#include <vector>

int main(int argc, char** argv) {
  const int64_t N = 1 << 20, B = 1024, A = 1024;
  const int piv[10] = {0, 1, 2, 4, 5, 7, 8, 11, 12, 14};
  std::vector<int64_t> off(A);
  for (int a = 0; a < A; ++a) {
    int64_t o = 0;
    for (int i = 0; i < 10; ++i) if ((a >> i) & 1) o += 1 << (20 - 1 - piv[i]);
    off[a] = o;
  }
  uint64_t* sig = (uint64_t*)aligned_alloc(1 << 21, sizeof(uint64_t) * N * B);
  const int nohuge = argc > 1 && argv[1][0] == 'n';
  madvise(sig, sizeof(uint64_t) * N * B, nohuge ? MADV_NOHUGEPAGE : MADV_HUGEPAGE);
  printf("pages: %s\n", nohuge ? "4K (MADV_NOHUGEPAGE)" : "THP requested");
#pragma omp parallel for
  for (int64_t i = 0; i < N * B; ++i) sig[i] = i;
  uint64_t* out = (uint64_t*)aligned_alloc(4096, sizeof(uint64_t) * B * A);
  const int thr_list[] = {16};
  const int dist_list[] = {0, 4, 8, 16, 32};
  for (int nt : thr_list) {
   for (int hint = 0; hint < 4; ++hint) {
    for (int D : dist_list) {
      if (D == 0 && hint) continue;
      double best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(nt)
        {
          const int w = omp_get_thread_num(), nw = omp_get_num_threads();
          const int64_t per = (B + nw - 1) / nw, b0 = w * per, b1 = std::min(B, b0 + per);
          const int64_t i0 = b0 * A, i1 = b1 * A;
          if (D == 0) {
            for (int64_t i = i0; i < i1; ++i) out[i] = sig[(i / A) * N + off[i % A]];
          } else {
            for (int64_t i = i0; i < i1; ++i) {
              const int64_t j = i + D;
              if (j < i1) {
                const uint64_t* q = sig + (j / A) * N + off[j % A];
                if (hint == 0) __builtin_prefetch(q, 0, 0);
                else if (hint == 1) __builtin_prefetch(q, 0, 1);
                else if (hint == 2) __builtin_prefetch(q, 0, 2);
                else __builtin_prefetch(q, 0, 3);
              }
              out[i] = sig[(i / A) * N + off[i % A]];
            }
          }
        }
        auto t1 = std::chrono::steady_clock::now();
        best = std::min(best, std::chrono::duration<double, std::milli>(t1 - t0).count());
      }
      printf("threads %2d prefetch locality-hint %d distance %2d: %.3f ms\n", nt, hint, D, best);
    }
   }
  }
  return (int)(out[12345] & 1);
}
