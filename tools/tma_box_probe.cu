// TMA box-size probe for the head pass (config 5 pattern, 16 B pieces):
// (a) 512-row boxes: four run dims (row index folded into dim 4 with the
//     q2..q4 run), 8 ops per unit;  (b) 128-row boxes: three run dims and
//     the row in dim 4 (the head's map), 32 ops per unit.  Same bytes.
// One CTA of 128 threads per (row, piece); thread 0 issues, all wait.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(128) k(const __grid_constant__ CUtensorMap tm, int rows, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  constexpr int C = 8, PIECE = 2;
  const int row = blockIdx.x / C, c = blockIdx.x % C;
  constexpr uint32_t BYTES = 4096u * PIECE * 8u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(saddr(&mbar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(saddr(&mbar)), "r"(BYTES) : "memory");
    constexpr int OPS = MODE == 0 ? 8 : 32;
    for (int op = 0; op < OPS; ++op) {
      int c0, c1, c2, c3, c4;
      const uint32_t dst = saddr(sm + op * (BYTES / OPS));
      if (MODE == 0) {  // dims: 256 | 16 (q10,q9) | 8 (q8,q7) | 8 (q6,q5) | rows<<8 (q4..q2 + high)
        const int64_t base = (int64_t)c * PIECE + ((op & 1) ? (1 << 25) : 0) + ((op & 2) ? (1 << 23) : 0) + ((op & 4) ? 64 : 0);
        c0 = (int)(base & 255); c1 = (int)((base >> 8) & 15); c2 = (int)((base >> 12) & 7); c3 = (int)((base >> 15) & 7);
        c4 = (int)((base >> 18) + ((int64_t)row << 8));
      } else {  // head map: dim0 [0,8) bits, dim1 [8,12), dim2 [12,18), dim3 [18,26), dim4 rows; leftover q0,q1,q5,q6,q11
        uint32_t e = (uint32_t)c * PIECE;
        if (op & 1) e += 1u << 25;
        if (op & 2) e += 1u << 23;
        if (op & 4) e += 1u << 16;
        if (op & 8) e += 1u << 15;
        if (op & 16) e += 64;
        c0 = (int)(e & 255); c1 = (int)((e >> 8) & 15); c2 = (int)((e >> 12) & 63); c3 = (int)(e >> 18); c4 = row;
      }
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          :: "r"(dst), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(saddr(&mbar)) : "memory");
    }
  }
  __syncthreads();
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(saddr(&mbar)) : "memory");
  const float acc = reinterpret_cast<float*>(sm)[threadIdx.x];
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const int rows = 128;
  const int64_t ld = 1ll << 26;
  float2* sig;
  if (cudaMalloc(&sig, (size_t)rows * ld * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(sig, 0, (size_t)rows * ld * 8);
  float* sink;
  cudaMalloc(&sink, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  for (int mode = 0; mode < 2; ++mode) {
    CUtensorMap tm;
    CUresult r;
    if (mode == 0) {
      cuuint64_t dims[5] = {256, 16, 8, 8, (cuuint64_t)rows << 8};
      cuuint64_t strides[4] = {256 * 8ull, 4096 * 8ull, 32768 * 8ull, 262144 * 8ull};
      cuuint32_t box[5] = {2, 4, 4, 4, 8};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 5, sig, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t dims[5] = {256, 16, 64, 256, (cuuint64_t)rows};
      cuuint64_t strides[4] = {256 * 8ull, 4096 * 8ull, 262144 * 8ull, (cuuint64_t)ld * 8};
      cuuint32_t box[5] = {2, 4, 4, 8, 1};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 5, sig, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    auto kern = mode == 0 ? k<0> : k<1>;
    const int smem = 4096 * 2 * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<rows * 8, 128, smem>>>(tm, rows, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) kern<<<rows * 8, 128, smem>>>(tm, rows, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s): %.3f ms/launch  %.1f GB/s of line bytes  [%s]\n", mode,
           mode == 0 ? "512-row boxes, 8 ops" : "128-row boxes, 32 ops", ms / 5,
           (double)rows * 4096 * 128 * 5 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
