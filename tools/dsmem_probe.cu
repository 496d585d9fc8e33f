// DSMEM bandwidth probe: clusters of C CTAs, each CTA moves its 32 KB slice to
// the other CTAs of its cluster by different access patterns.
//   V0 st.async 8B, scattered (owner = low bits of the index: every lane a different CTA)
//   V1 st.async 16B, contiguous blocks (lanes write consecutive 16B of one destination)
//   V2 remote ld 8B contiguous   (generic pointer from map_shared_rank)
//   V3 remote ld 16B contiguous
//   V4 plain remote st 16B contiguous + cluster barrier
//   V5 global (L2) exchange: coalesced 16B store to scratch, cluster barrier, coalesced 16B load
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int C = 16, NT = 256, SL = 2048;  // 2048 c64 = 16 KB per CTA

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}

template <int V>
__global__ void __launch_bounds__(NT) k(float2* scratch, float* sink, int iters) {
  __shared__ __align__(16) float2 buf[SL];
  __shared__ __align__(16) float2 rcv[SL];
  __shared__ __align__(8) unsigned long long mbar;
  cg::cluster_group cl = cg::this_cluster();
  const int q = cl.block_rank(), t = threadIdx.x;
  for (int i = t; i < SL; i += NT) buf[i] = make_float2(i, q);
  const uint32_t mb = saddr(&mbar);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    if (V == 0 || V == 1) {
      if (t == 0) asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(SL * 8) : "memory");
      cl.sync();
      if (V == 0) {
        for (int i = t; i < SL; i += NT) {
          const uint32_t owner = i & (C - 1);
          const uint32_t pos = (i >> 4) + q * (SL / C);
          const uint32_t dst = mapa(saddr(&rcv[pos]), owner);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                       :: "r"(dst), "f"(buf[i].x), "f"(buf[i].y), "r"(mapa(mb, owner)) : "memory");
        }
      } else {
        // 16B: owner block r gets SL/C contiguous elements = 128 x 16B
        for (int j = t; j < SL / 2; j += NT) {
          const int r = j / (SL / C / 2), w = j % (SL / C / 2);
          const float4 v = reinterpret_cast<const float4*>(buf)[j];
          const uint32_t dst = mapa(saddr(&rcv[q * (SL / C) + 2 * w]), r);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                       :: "r"(dst), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mapa(mb, r)) : "memory");
        }
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mb), "r"(it & 1) : "memory");
      acc += rcv[t].x;
    } else if (V == 2 || V == 3) {
      cl.sync();
      for (int r = 0; r < C; ++r) {
        const float2* rem = cl.map_shared_rank(buf, r);
        if (V == 2) {
          for (int i = t; i < SL / C; i += NT) acc += rem[q * (SL / C) + i].x;
        } else {
          const float4* r4 = reinterpret_cast<const float4*>(rem + q * (SL / C));
          for (int i = t; i < SL / C / 2; i += NT) acc += r4[i].x;
        }
      }
    } else if (V == 4) {
      for (int r = 0; r < C; ++r) {
        float4* rem = reinterpret_cast<float4*>(cl.map_shared_rank(rcv, r) + q * (SL / C));
        const float4* src = reinterpret_cast<const float4*>(buf + r * (SL / C));
        for (int i = t; i < SL / C / 2; i += NT) rem[i] = src[i];
      }
      cl.sync();
      acc += rcv[t].x;
    } else if (V == 5) {
      float4* sc = reinterpret_cast<float4*>(scratch) + (size_t)(blockIdx.x / C) * C * SL / 2;
      for (int r = 0; r < C; ++r) {
        const float4* src = reinterpret_cast<const float4*>(buf + r * (SL / C));
        for (int i = t; i < SL / C / 2; i += NT) sc[(r * C + q) * (SL / C / 2) + i] = src[i];
      }
      cl.sync();
      for (int x = 0; x < C; ++x)
        for (int i = t; i < SL / C / 2; i += NT) acc += sc[(q * C + x) * (SL / C / 2) + i].x;
      cl.sync();
    }
  }
  cl.sync();
  if (acc == 12345.f) sink[0] = acc;
}

template <int V>
float run(int grid, float2* scratch, float* sink, int iters) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchKernelEx(&cfg, k<V>, scratch, sink, 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k<V>, scratch, sink, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("V%d status %s\n", V, cudaGetErrorString(cudaGetLastError()));
  return ms;
}

int main() {
  const int grid = 148 / C * C * 4;  // ~4 CTAs per SM worth of clusters
  const int iters = 200;
  float2* scratch;
  float* sink;
  cudaMalloc(&scratch, (size_t)grid * SL * 8);
  cudaMalloc(&sink, 4);
  const double bytes = (double)grid * SL * 8 * (C - 1) / C * iters;  // remote bytes moved
  const char* names[] = {"st.async 8B scattered", "st.async 16B blocks", "remote ld 8B contig", "remote ld 16B contig",
                         "remote st 16B + cluster.sync", "global L2 exchange 16B"};
  float ms[6];
  ms[0] = run<0>(grid, scratch, sink, iters);
  ms[1] = run<1>(grid, scratch, sink, iters);
  ms[2] = run<2>(grid, scratch, sink, iters);
  ms[3] = run<3>(grid, scratch, sink, iters);
  ms[4] = run<4>(grid, scratch, sink, iters);
  ms[5] = run<5>(grid, scratch, sink, iters);
  for (int v = 0; v < 6; ++v)
    printf("%-30s %8.3f ms  %8.1f GB/s aggregate remote traffic (%d CTAs, %d iters)\n", names[v], ms[v],
           bytes / (ms[v] * 1e-3) / 1e9, grid, iters);
  return 0;
}
