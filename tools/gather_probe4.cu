// Probe: does DRAM page locality raise the isolated-line rate?  1M isolated
// 8 B samples (one per 128 B line) from 1024 rows 8 MiB apart, in layouts:
//   0 uniform: one line every 8 KiB
//   1 clusters of 8 adjacent lines (1 KiB), clusters 64 KiB apart
//   2 clusters of 16 lines every other line (4 KiB window), 128 KiB apart
//   3 the config-2 pattern (pivots 0 1 2 4 5 7 8 11 12 14 of M = 20), sorted
// Each thread loads 16 samples (consecutive pattern indices), 8 rotating
// row sets so L2 never hits.  Timed with events over 50 launches.
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) k_gather(const float2* __restrict__ sig, long ld_row, int rows,
                                                const int* __restrict__ offs, int A, long shift,
                                                float2* __restrict__ out) {
  const int tpr = A / 16;
  const long gid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long row = gid / tpr;
  const int t = gid % tpr;
  if (row >= rows) return;
  const float2* base = sig + row * ld_row + shift;
  float2 v[16];
#pragma unroll
  for (int x = 0; x < 16; ++x)
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y)
                 : "l"(base + offs[t * 16 + x]));
  float2 s = {0.f, 0.f};
#pragma unroll
  for (int x = 0; x < 16; ++x) { s.x += v[x].x; s.y += v[x].y; }
  out[gid] = s;
}

int main() {
  const int rows = 1024, A = 1024;
  const long N = 1 << 20;
  float2* sig;
  cudaMalloc(&sig, sizeof(float2) * N * rows);
  cudaMemset(sig, 0, sizeof(float2) * N * rows);
  int* d_off;
  cudaMalloc(&d_off, sizeof(int) * A);
  float2* out;
  cudaMalloc(&out, sizeof(float2) * rows * A / 16);
  const char* names[] = {"uniform 8 KiB stride", "clusters of 8 adjacent lines", "clusters of 16 alternate lines",
                         "config-2 pattern (sorted)", "config-2 pattern, slot order"};
  for (int layout = 0; layout < 5; ++layout) {
    std::vector<int> h(A);
    for (int q = 0; q < A; ++q) {
      if (layout == 0) h[q] = q * (int)(N / A);
      if (layout == 1) h[q] = (q / 8) * 8192 + (q % 8) * 16;        // elements: 64 KiB clusters, 128 B apart
      if (layout == 2) h[q] = (q / 16) * 16384 + (q % 16) * 32;     // 128 KiB clusters, 256 B apart
      if (layout >= 3) {
        const int piv[10] = {0, 1, 2, 4, 5, 7, 8, 11, 12, 14};
        int o = 0;
        for (int i = 0; i < 10; ++i)
          if ((q >> i) & 1) o += 1 << (19 - piv[i]);
        h[q] = o;
      }
    }
    if (layout == 3) std::sort(h.begin(), h.end());
    cudaMemcpy(d_off, h.data(), sizeof(int) * A, cudaMemcpyHostToDevice);
    const int grid = rows * (A / 16) / 256;
    for (int i = 0; i < 3; ++i) k_gather<<<grid, 256>>>(sig, N, rows, d_off, A, 16 * (i % 8), out);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 50; ++i) k_gather<<<grid, 256>>>(sig, N, rows, d_off, A, 16 * (i % 8), out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-34s %7.2f us per 1M lines (%.2e lines/s)\n", names[layout], ms * 1e3 / 50, 1.048576e6 / (ms * 1e-3 / 50));
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
