// Probe 2: what does one isolated sample cost in DRAM bytes, by access path?
//   V0  ld.global.nc.L1::no_allocate.v2.f32     (8 B, read-only path)
//   V1  ld.global.f32 x1                         (4 B)
//   V2  ld.global.nc.v4.f32                      (16 B)
//   V3  cp.async.ca.shared.global 8 B            (LDGSTS)
//   V4  cp.async.bulk 16 B -> smem (TMA engine, mbarrier)
//   V5  ld.global.nc.L1::no_allocate.L2::evict_first.v2.f32
// Same gather pattern as config 2: 1024 rows x 1024 samples, one per 128B line.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

template <int V>
__global__ void __launch_bounds__(256) k_probe(const float2* __restrict__ sig, long ld_row, int rows,
                                               const int* __restrict__ offs, int A, int shift,
                                               float2* __restrict__ out) {
  constexpr int E = 16;
  __shared__ __align__(16) float4 stage[256 * E / 2];
  __shared__ __align__(8) unsigned long long mbar;
  const int tpr = A / E;
  const long gid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const long row = gid / tpr;
  const int t = gid % tpr;
  const bool live = row < rows;
  const float2* base = sig + (live ? row : 0) * ld_row + shift;
  float sx = 0.f, sy = 0.f;
  if (V == 0 || V == 1 || V == 2 || V == 5 || V == 6 || V == 7) {
    float2 v[E];
#pragma unroll
    for (int x = 0; x < E; ++x) {
      const float2* p = base + offs[t * E + x];
      if (V == 0) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y) : "l"(p));
      if (V == 5) asm volatile("{ .reg .b64 pol; createpolicy.fractional.L2::evict_first.b64 pol, 1.0; ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], pol; }" : "=f"(v[x].x), "=f"(v[x].y) : "l"(p));
      if (V == 6) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y) : "l"(p));
      if (V == 7) asm volatile("ld.global.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v[x].x), "=f"(v[x].y) : "l"(p));
      if (V == 1) { asm volatile("ld.global.f32 %0, [%1];" : "=f"(v[x].x) : "l"(p)); v[x].y = 0.f; }
      if (V == 2) {
        const float4* q = reinterpret_cast<const float4*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15);
        float4 w;
        asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w) : "l"(q));
        v[x].x = w.x + w.z; v[x].y = w.y + w.w;
      }
    }
#pragma unroll
    for (int x = 0; x < E; ++x) { sx += v[x].x; sy += v[x].y; }
  } else if (V == 3) {
    float2* st = reinterpret_cast<float2*>(stage) + threadIdx.x * E;
#pragma unroll
    for (int x = 0; x < E; ++x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_u32(st + x)), "l"(base + offs[t * E + x]));
    asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
    for (int x = 0; x < E; ++x) { sx += st[x].x; sy += st[x].y; }
  } else if (V == 4) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    constexpr int H = E / 2;
    for (int round = 0; round < 2; ++round) {
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(smem_u32(&mbar)), "r"(256 * H * 16));
      __syncthreads();
      float4* st = stage + threadIdx.x * H;
#pragma unroll
      for (int x = 0; x < H; ++x) {
        const float2* p = base + offs[t * E + round * H + x];
        const void* q = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                     :: "r"(smem_u32(st + x)), "l"(q), "r"(smem_u32(&mbar)) : "memory");
      }
      unsigned done = 0;
      while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&mbar)), "r"(round & 1) : "memory");
      }
#pragma unroll
      for (int x = 0; x < H; ++x) { sx += st[x].x + st[x].z; sy += st[x].y + st[x].w; }
      __syncthreads();
    }
  }
  if (live) out[gid] = make_float2(sx, sy);
}

template <int V>
float run(const float2* sig, long ld_row, int rows, const int* offs, int A, float2* out, int reps) {
  const long threads = (long)rows * (A / 16);
  const int grid = (int)((threads + 255) / 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_probe<V><<<grid, 256>>>(sig, ld_row, rows, offs, A, 16 * (i % 8), out);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_probe<V><<<grid, 256>>>(sig, ld_row, rows, offs, A, 16 * (i % 8), out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main(int argc, char** argv) {
  const int rows = 1024, A = 1024;
  const long N = 1 << 20;
  if (argc > 1) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(argv[1]));
    printf("fetch granularity %s: %s\n", argv[1], cudaGetErrorString(e));
  }
  float2* sig;
  cudaMalloc(&sig, sizeof(float2) * N * rows);
  cudaMemset(sig, 0, sizeof(float2) * N * rows);
  std::vector<int> h(A);
  srand(7);
  for (int q = 0; q < A; ++q) h[q] = q * (int)(N / A) + (rand() % 8) * 2 % 16;
  int* offs;
  cudaMalloc(&offs, sizeof(int) * A);
  cudaMemcpy(offs, h.data(), sizeof(int) * A, cudaMemcpyHostToDevice);
  float2* out;
  cudaMalloc(&out, sizeof(float2) * rows * A);
  const int reps = 50;
  const char* names[] = {"ldg.nc 8B", "ldg 4B", "ldg.nc 16B", "cp.async 8B", "tma bulk 16B", "ldg.nc evict_first", "ldg.nc L2::64B", "ldg L2::64B"};
  float t[8];
  t[0] = run<0>(sig, N, rows, offs, A, out, reps);
  t[1] = run<1>(sig, N, rows, offs, A, out, reps);
  t[2] = run<2>(sig, N, rows, offs, A, out, reps);
  t[3] = run<3>(sig, N, rows, offs, A, out, reps);
  t[4] = run<4>(sig, N, rows, offs, A, out, reps);
  t[5] = run<5>(sig, N, rows, offs, A, out, reps);
  t[6] = run<6>(sig, N, rows, offs, A, out, reps);
  t[7] = run<7>(sig, N, rows, offs, A, out, reps);
  for (int v = 0; v < 8; ++v)
    printf("%-20s %8.2f us  %.3e samples/s\n", names[v], t[v], rows * (double)A / (t[v] * 1e-6));
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
