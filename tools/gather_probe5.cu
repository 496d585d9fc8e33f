// Probe: isolated-line gather rate vs loads in flight per thread (E) and
// CTA size, config-2 pattern (1024 rows x 1024 samples, rows 8 MiB apart).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

template <int E>
__global__ void k_gather(const float2* __restrict__ sig, long ld_row, int rows, const int* __restrict__ offs,
                         int A, long shift, float2* __restrict__ out) {
  const int tpr = A / E;
  const long gid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long row = gid / tpr;
  const int t = gid % tpr;
  if (row >= rows) return;
  const float2* base = sig + row * ld_row + shift;
  float2 v[E];
#pragma unroll
  for (int x = 0; x < E; ++x)
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y)
                 : "l"(base + offs[t * E + x]));
  float2 s = {0.f, 0.f};
#pragma unroll
  for (int x = 0; x < E; ++x) { s.x += v[x].x; s.y += v[x].y; }
  out[gid] = s;
}

template <int E>
void run(const float2* sig, long N, int rows, const int* d_off, int A, float2* out, int nt) {
  const long threads = (long)rows * (A / E);
  const int grid = (int)((threads + nt - 1) / nt);
  for (int i = 0; i < 3; ++i) k_gather<E><<<grid, nt>>>(sig, N, rows, d_off, A, 16 * (i % 8), out);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 50; ++i) k_gather<E><<<grid, nt>>>(sig, N, rows, d_off, A, 16 * (i % 8), out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("E=%2d CTA=%4d: %7.2f us per 1M lines (%.2e lines/s)\n", E, nt, ms * 1e3 / 50, 1.048576e6 / (ms * 1e-3 / 50));
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
  cudaMalloc(&out, sizeof(float2) * rows * A);
  std::vector<int> h(A);
  const int piv[10] = {0, 1, 2, 4, 5, 7, 8, 11, 12, 14};
  for (int q = 0; q < A; ++q) {
    int o = 0;
    for (int i = 0; i < 10; ++i)
      if ((q >> i) & 1) o += 1 << (19 - piv[i]);
    h[q] = o;
  }
  cudaMemcpy(d_off, h.data(), sizeof(int) * A, cudaMemcpyHostToDevice);
  for (int nt : {64, 128, 256, 512}) {
    run<4>(sig, N, rows, d_off, A, out, nt);
    run<8>(sig, N, rows, d_off, A, out, nt);
    run<16>(sig, N, rows, d_off, A, out, nt);
    run<32>(sig, N, rows, d_off, A, out, nt);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
