// Load-pattern probe for the cluster transform (config 5): C CTAs per row
// each read one 32 B (C=4) / 16 B (C=8) piece of every 128 B line the row's
// sample set touches (4096 lines per row at the config-5 pivots), so the C
// CTAs of a row together read every line once.  Variants:
//   ldg   : LDG.128 into registers (summed)
//   cpasync: cp.async 16 B into shared memory (one row slice per CTA)
// rows are spread over a buffer larger than L2; CTAs of one row are adjacent
// block indices (they run concurrently, so a line fetched by one is an L2 hit
// for the others).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 26;
__constant__ uint32_t d_off[12];  // stride of q bits 0..11 (elements)

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int C, int V>
__global__ void __launch_bounds__(512) k(const float2* __restrict__ sig, int64_t ld, int rows, float* sink) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int PIECE = 16 / C;            // elements per CTA per line (4 or 2)
  constexpr int V16 = PIECE / 2;           // 16 B vectors per line per CTA
  const int row = blockIdx.x / C, c = blockIdx.x % C;
  if (row >= rows) return;
  const float2* base = sig + (int64_t)row * ld + c * PIECE;
  float acc = 0.f;
  // thread t handles q = t + 512 n
  for (int n = 0; n < 4096 / 512; ++n) {
    const uint32_t qv = threadIdx.x + 512 * n;
    uint32_t o = 0;
#pragma unroll
    for (int i = 0; i < 12; ++i)
      if ((qv >> i) & 1) o += d_off[i];
#pragma unroll
    for (int v = 0; v < V16; ++v) {
      const float4* p = reinterpret_cast<const float4*>(base + o) + v;
      if (V == 0) {
        float4 x;
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "l"(p));
        acc += x.x + x.w;
      } else {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(saddr(sm + ((qv * V16 + v) * 16))), "l"(p) : "memory");
      }
    }
  }
  if (V == 1) {
    asm volatile("cp.async.commit_group; cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    acc = reinterpret_cast<float*>(sm)[threadIdx.x];
  }
  if (acc == 12345.f) sink[0] = acc;
}

template <int C, int V>
void run(const char* name, const float2* sig, int64_t ld, int rows, float* sink) {
  auto kern = k<C, V>;
  const int smem = V ? 4096 * 16 * (16 / C / 2) : 0;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<rows * C, 512, smem>>>(sig, ld, rows, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<rows * C, 512, smem>>>(sig, ld, rows, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)rows * 4096 * 128 * reps;
  printf("%-10s C=%d rows=%d  %.3f ms/launch  %.1f GB/s of line bytes  [%s]\n", name, C, rows, ms / reps,
         bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int piv[16] = {0, 2, 5, 6, 7, 9, 10, 12, 13, 16, 17, 19, 22, 23, 24, 25};
  uint32_t off[12];
  for (int i = 0; i < 12; ++i) off[i] = 1u << (M - 1 - piv[i]);
  cudaMemcpyToSymbol(d_off, off, sizeof(off));
  const int rows = 128;
  const int64_t ld = 1ll << M;
  float2* sig;
  if (cudaMalloc(&sig, (size_t)rows * ld * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(sig, 0, (size_t)rows * ld * 8);
  float* sink;
  cudaMalloc(&sink, 4);
  run<4, 0>("ldg", sig, ld, rows, sink);
  run<4, 1>("cpasync", sig, ld, rows, sink);
  run<8, 0>("ldg", sig, ld, rows, sink);
  run<8, 1>("cpasync", sig, ld, rows, sink);
  run<1, 0>("ldg", sig, ld, rows, sink);
  return 0;
}
