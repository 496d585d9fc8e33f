// DSMEM throughput probe for the cluster transform design (config 5):
// clusters of C CTAs, each CTA holds BYTES of data in shared memory and
// every CTA pulls 1/C of every CTA's buffer (16 B remote loads,
// ld.shared::cluster.v4) -- the final-phase exchange pattern.  Variants:
//   pull+bar : pull, then a cluster barrier per iteration (arrive.release / wait.acquire)
//   pull     : pull only (no barrier; throughput ceiling)
//   push     : st.async 16 B with mbarrier complete_tx, wait per iteration
// Reports aggregate remote bytes/s and bytes per SM clock.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t cl_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int C, int NT, int BYTES, int V>
__global__ void __launch_bounds__(NT) k(float* sink, int iters) {
  extern __shared__ __align__(16) unsigned char sm[];
  float4* buf = reinterpret_cast<float4*>(sm);
  float4* rcv = reinterpret_cast<float4*>(sm + BYTES);
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(sm + 2 * BYTES);
  const uint32_t q = cl_rank();
  const int t = threadIdx.x;
  constexpr int N16 = BYTES / 16, PER = N16 / C;  // 16 B words per CTA, pulled per CTA from each peer
  for (int i = t; i < N16; i += NT) buf[i] = make_float4(i, q, 1, 2);
  if (V == 2 && t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(saddr(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl_sync();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    if (V < 2) {
#pragma unroll 4
      for (int j = t; j < PER; j += NT) {
#pragma unroll
        for (int r = 0; r < C; ++r) {
          const uint32_t src = (q + r) % C;
          const uint32_t a = mapa(saddr(buf + q * PER + j), src);
          float4 v;
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
          acc += v.x + v.w;
        }
      }
      if (V == 0) cl_sync();
    } else {
      if (t == 0)
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(saddr(mbar)), "r"(BYTES) : "memory");
      cl_sync();
      for (int j = t; j < PER; j += NT) {
#pragma unroll
        for (int r = 0; r < C; ++r) {
          const uint32_t dst = (q + r) % C;
          const float4 v = buf[dst * PER + j];
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                       :: "r"(mapa(saddr(rcv + q * PER + j), dst)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w),
                          "r"(mapa(saddr(mbar), dst)) : "memory");
        }
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(saddr(mbar)), "r"(it & 1) : "memory");
      acc += reinterpret_cast<float*>(rcv)[t];
    }
  }
  cl_sync();
  if (acc == 12345.f) sink[0] = acc;
}

template <int C, int NT, int BYTES, int V>
void run(const char* name, int extra_smem) {
  auto kern = k<C, NT, BYTES, V>;
  const size_t smem = 2 * BYTES + 64 + extra_smem;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int ncl = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (e != cudaSuccess || ncl == 0) { printf("%s: occupancy error %s\n", name, cudaGetErrorString(e)); return; }
  cfg.gridDim = dim3(C * ncl);
  float* sink;
  cudaMalloc(&sink, 4);
  cudaLaunchKernelEx(&cfg, kern, sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 200;
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, sink, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  e = cudaGetLastError();
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double remote = (double)C * ncl * BYTES * (C - 1) / C * iters;
  const int ctas = C * ncl;
  printf("%-34s C=%d NT=%d %3d KB/CTA clusters=%3d CTAs=%3d  %7.3f ms  %7.1f GB/s remote  %5.1f B/clk/CTA  [%s]\n", name, C, NT,
         BYTES / 1024, ncl, ctas, ms, remote / (ms * 1e-3) / 1e9,
         remote / ctas / (ms * 1e-3 * clk * 1e3), cudaGetErrorString(e));
  cudaFree(sink);
}

int main() {
  run<4, 512, 65536 * 2, 0>("pull+bar 128KB", 0);
  run<4, 512, 65536 * 2, 1>("pull 128KB", 0);
  run<4, 512, 65536 * 2 / 2, 2>("push 64KB", 0);
  run<8, 512, 65536, 0>("pull+bar 64KB 1/SM", 32768);
  run<8, 512, 65536, 1>("pull 64KB 1/SM", 32768);
  run<8, 512, 65536, 2>("push 64KB 1/SM", 32768);
  run<8, 256, 32768, 0>("pull+bar 32KB 2/SM?", 0);
  run<8, 256, 32768, 1>("pull 32KB 2/SM?", 0);
  run<8, 256, 32768, 2>("push 32KB 2/SM?", 0);
  run<2, 512, 65536 * 2, 0>("pull+bar C2 128KB", 0);
  run<16, 256, 32768, 1>("pull C16 32KB", 0);
  return 0;
}
