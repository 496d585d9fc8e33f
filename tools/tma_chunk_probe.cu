// TMA probe for the config-5 gather: one rank-5 tensor map over a row
// (dim0 = the CTA's piece of a 128 B line, dims 1-4 = runs of consecutive
// pivots) loads 512 lines' pieces per cp.async.bulk.tensor; a CTA issues the
// ops for its (row, piece) and waits on one mbarrier.  Compared with
// cp.async 16 B per thread on the same pattern.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 26;
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// q bits: run dims (q2..q4 -> stride 2^18 size 8), (q9,q10 -> 2^8 size 4 : q10 stride 256, q9 512),
// (q7,q8 -> 2^12 size 4), (q5,q6 -> 2^15 size 4); remaining q0 (2^25), q1 (2^23), q11 (2^6) by ops
template <int PIECE>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap tm, int rows, float* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  constexpr int C = 16 / PIECE;
  const int row = blockIdx.x / C, c = blockIdx.x % C;
  if (row >= rows) return;
  constexpr uint32_t BYTES = 4096u * PIECE * 8u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(saddr(&mbar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(saddr(&mbar)), "r"(BYTES) : "memory");
    for (int op = 0; op < 8; ++op) {
      // coordinates: dim0 = element index within the row base (c*PIECE + q0,q1,q11 offsets folded in dim0? no: use dim0 start)
      const int64_t base = (int64_t)c * PIECE + ((op & 1) ? (1 << 25) : 0) + ((op & 2) ? (1 << 23) : 0) + ((op & 4) ? 64 : 0);
      // dims: 0 elements (stride 1), 1 run q10q9 (stride 256), 2 run q8q7 (4096), 3 run q6q5 (2^15), 4 run q4q3q2 (2^18 x row)
      // dim0 spans the whole row; the row index lives in dim4's extent
      const int c0 = (int)(base & ((1 << 8) - 1));  // within 256
      const int c1 = (int)((base >> 8) & 15), c2 = (int)((base >> 12) & 7), c3 = (int)((base >> 15) & 7);
      const int c4 = (int)((base >> 18) + ((int64_t)row << 8));
      const uint32_t dst = saddr(sm + op * (BYTES / 8));
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
  const int64_t ld = 1ll << M;
  float2* sig;
  if (cudaMalloc(&sig, (size_t)rows * ld * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(sig, 0, (size_t)rows * ld * 8);
  float* sink;
  cudaMalloc(&sink, 4);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  for (int PIECE : {4, 2}) {
    // view the whole buffer as [rows*2^8][8][8][16][256] of 8 B elements (strides 2^18, 2^15, 2^12, 2^8, 1)
    // and take boxes {PIECE, 4 (q10,q9 at 256,512), 4 (q8,q7), 4 (q6,q5), 8 (q4..q2)}
    cuuint64_t dims[5] = {256, 16, 8, 8, (cuuint64_t)rows << 8};
    cuuint64_t strides[4] = {256 * 8ull, 4096 * 8ull, 32768 * 8ull, 262144 * 8ull};
    // box strides via elementStrides: dim1 step 1 of stride 256 -> q10 (256) and q9 (512): box 4 with elementStride 1
    cuuint32_t box[5] = {(cuuint32_t)PIECE, 4, 4, 4, 8};
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUtensorMap tm;
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 5, sig, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    const int C = 16 / PIECE;
    const int smem = 4096 * PIECE * 8;
    auto kern = PIECE == 4 ? k_tma<4> : k_tma<2>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<rows * C, 128, smem>>>(tm, rows, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 5;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) kern<<<rows * C, 128, smem>>>(tm, rows, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("tma piece=%d C=%d rows=%d  %.3f ms/launch  %.1f GB/s of line bytes  [%s]\n", PIECE, C, rows, ms / reps,
           (double)rows * 4096 * 128 * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
