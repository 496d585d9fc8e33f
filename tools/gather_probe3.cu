// Probe 3: config-2 sample pattern, slot order vs sorted-address order per
// warp (DRAM row locality), 1024 rows x 1024 samples, rotating 8 row sets.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

template <int ORDER>  // 0: slot order (x + t*16 as the product kernel), 1: sorted order per thread block
__global__ void __launch_bounds__(64) k(const float2* __restrict__ sig, long ld, const int* __restrict__ offs_slot,
                                        const int* __restrict__ offs_sorted, float2* __restrict__ out, int set) {
  const int t = threadIdx.x, b = blockIdx.x;
  const float2* row = sig + ((long)b + (long)set * 1024) * ld;
  float2 v[16];
#pragma unroll
  for (int x = 0; x < 16; ++x) {
    const int o = ORDER == 0 ? offs_slot[x + t * 16] : offs_sorted[t + x * 64];
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y) : "l"(row + o));
  }
  float2 s = {0, 0};
#pragma unroll
  for (int x = 0; x < 16; ++x) { s.x += v[x].x; s.y += v[x].y; }
  out[b * 64 + t] = s;
}

int main() {
  const int M = 20, A = 1024;
  const int piv[10] = {0, 1, 2, 4, 5, 7, 8, 11, 12, 14};  // config 2 pivots
  std::vector<int> slot(A), sorted(A);
  for (int a = 0; a < A; ++a) {
    int off = 0;
    for (int i = 0; i < 10; ++i) if ((a >> i) & 1) off += 1 << (M - 1 - piv[i]);
    slot[a] = off;
  }
  sorted = slot;
  std::sort(sorted.begin(), sorted.end());
  const long N = 1 << M, sets = 4;
  float2* sig;
  cudaMalloc(&sig, sizeof(float2) * N * 1024 * sets);
  cudaMemset(sig, 0, sizeof(float2) * N * 1024 * sets);
  int *ds, *dq;
  cudaMalloc(&ds, 4 * A);
  cudaMalloc(&dq, 4 * A);
  cudaMemcpy(ds, slot.data(), 4 * A, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, sorted.data(), 4 * A, cudaMemcpyHostToDevice);
  float2* out;
  cudaMalloc(&out, sizeof(float2) * 1024 * 64);
  for (int order = 0; order < 2; ++order) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 8; ++i) {
      if (order == 0) k<0><<<1024, 64>>>(sig, N, ds, dq, out, i % sets);
      else k<1><<<1024, 64>>>(sig, N, ds, dq, out, i % sets);
    }
    cudaEventRecord(a);
    for (int i = 0; i < 100; ++i) {
      if (order == 0) k<0><<<1024, 64>>>(sig, N, ds, dq, out, i % sets);
      else k<1><<<1024, 64>>>(sig, N, ds, dq, out, i % sets);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s order: %.2f us per 1M-sample gather\n", order ? "sorted" : "slot", ms * 10);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
