// L2 streaming bandwidth: a buffer that fits L2 (footprint F) written then
// read back with coalesced 16 B accesses by a full grid, timed with events
// (median of reps).  Also the same with a footprint well above L2 (HBM).
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__global__ void k_write(float4* p, size_t n, float v) {
  for (int r = 0; r < 8; ++r)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(v, v, v, v);
}
__global__ void k_read(const float4* p, size_t n, float* sink) {
  float acc = 0.f;
  for (int r = 0; r < 8; ++r)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 x = p[i];
    acc += x.x + x.w;
  }
  if (acc == 123.f) sink[0] = acc;
}
__global__ void k_copy(const float4* a, float4* b, size_t n) {
  for (int r = 0; r < 8; ++r)
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  const size_t sizes[] = {8u << 20, 16u << 20, 32u << 20, 48u << 20, 64u << 20, 1024u << 20};
  float4 *a, *b;
  cudaMalloc(&a, 1024u << 20);
  cudaMalloc(&b, 1024u << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8, nt = 256;
  for (size_t bytes : sizes) {
    const size_t n = bytes / 16;
    std::vector<float> tw, tr, tc;
    for (int rep = 0; rep < 9; ++rep) {
      float ms;
      k_read<<<grid, nt>>>(a, n, sink);  // warm (bring into L2)
      cudaEventRecord(e0);
      k_write<<<grid, nt>>>(a, n, (float)rep);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tw.push_back(ms);
      cudaEventRecord(e0);
      k_read<<<grid, nt>>>(a, n, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tr.push_back(ms);
      k_read<<<grid, nt>>>(b, n, sink);
      cudaEventRecord(e0);
      k_copy<<<grid, nt>>>(a, b, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      tc.push_back(ms);
    }
    std::sort(tw.begin(), tw.end());
    std::sort(tr.begin(), tr.end());
    std::sort(tc.begin(), tc.end());
    printf("x8 passes, footprint %5zu MiB: write %7.1f GB/s  read %7.1f GB/s  copy(r+w) %7.1f GB/s   (%.1f / %.1f / %.1f us)\n",
           bytes >> 20, 8 * bytes / (tw[4] * 1e-3) / 1e9, 8 * bytes / (tr[4] * 1e-3) / 1e9, 16 * bytes / (tc[4] * 1e-3) / 1e9,
           tw[4] * 1e3, tr[4] * 1e3, tc[4] * 1e3);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
