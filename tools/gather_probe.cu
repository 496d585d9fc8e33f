// Probe: isolated 8-byte gathers (one per 128B line) from an 8 GiB buffer,
// with different load flavours and L2 fetch granularities.  Answers how many
// DRAM bytes a lone 32B-sector access costs on this B200 and at what rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ float2 ld(const float2* p) {
  float2 r;
  if (V == 0) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 1) asm volatile("ld.global.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 2) asm volatile("ld.global.cg.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 3) asm volatile("ld.global.cs.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 4) asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 5) asm volatile("ld.global.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  if (V == 6) asm volatile("ld.global.relaxed.gpu.v2.f32 {%0,%1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// each thread gathers E samples of one row at offs[] + shift, sums them
template <int V, int E>
__global__ void __launch_bounds__(256) k_gather(const float2* __restrict__ sig, long ld_row, int rows,
                                                const int* __restrict__ offs, int A, int shift,
                                                float2* __restrict__ out) {
  const int tpr = A / E;
  const long gid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long row = gid / tpr;
  const int t = gid % tpr;
  if (row >= rows) return;
  const float2* base = sig + row * ld_row + shift;
  float2 v[E];
#pragma unroll
  for (int x = 0; x < E; ++x) v[x] = ld<V>(base + offs[t * E + x]);
  float2 s = {0.f, 0.f};
#pragma unroll
  for (int x = 0; x < E; ++x) { s.x += v[x].x; s.y += v[x].y; }
  out[gid] = s;
}

template <int V>
float run(const float2* sig, long ld_row, int rows, const int* offs, int A, float2* out, int reps) {
  const long threads = (long)rows * (A / 16);
  const int grid = (int)((threads + 255) / 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_gather<V, 16><<<grid, 256>>>(sig, ld_row, rows, offs, A, 16 * (i % 8), out);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_gather<V, 16><<<grid, 256>>>(sig, ld_row, rows, offs, A, 16 * (i % 8), out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main(int argc, char** argv) {
  const int rows = 1024, A = 1024;
  const long N = 1 << 20;
  const int gran = argc > 1 ? atoi(argv[1]) : -1;
  if (gran >= 0) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("set L2 fetch granularity %d -> %s, now %zu\n", gran, cudaGetErrorString(e), g);
  } else {
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    printf("default L2 fetch granularity %zu\n", g);
  }
  float2* sig;
  cudaMalloc(&sig, sizeof(float2) * N * rows);
  cudaMemset(sig, 0, sizeof(float2) * N * rows);
  // one sample per 128B line, lines spread over the row, random word in line
  std::vector<int> h(A);
  srand(7);
  for (int q = 0; q < A; ++q) h[q] = q * (int)(N / A) + (rand() % 8) * 2 % 16;
  int* offs;
  cudaMalloc(&offs, sizeof(int) * A);
  cudaMemcpy(offs, h.data(), sizeof(int) * A, cudaMemcpyHostToDevice);
  float2* out;
  cudaMalloc(&out, sizeof(float2) * rows * A);
  const int reps = 50;
  const char* names[] = {"nc.L1::no_allocate", "default", "cg", "cs", "nc", "L1::no_allocate", "relaxed.gpu"};
  float t[7];
  t[0] = run<0>(sig, N, rows, offs, A, out, reps);
  t[1] = run<1>(sig, N, rows, offs, A, out, reps);
  t[2] = run<2>(sig, N, rows, offs, A, out, reps);
  t[3] = run<3>(sig, N, rows, offs, A, out, reps);
  t[4] = run<4>(sig, N, rows, offs, A, out, reps);
  t[5] = run<5>(sig, N, rows, offs, A, out, reps);
  t[6] = run<6>(sig, N, rows, offs, A, out, reps);
  for (int v = 0; v < 7; ++v)
    printf("%-20s %8.2f us  %.3e samples/s  sector-GB/s %.0f\n", names[v], t[v], rows * (double)A / (t[v] * 1e-6),
           rows * (double)A * 32 / (t[v] * 1e-6) / 1e9);
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
