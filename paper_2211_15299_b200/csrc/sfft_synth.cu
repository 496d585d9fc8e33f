// On-device synthesis of band-limited samples (reference core.py:129-177):
//   f(n) = (1/N) sum_{l in J} c_l e^{+2 pi i n l / N}
// at arbitrary locations, in float64 with the exponent reduced exactly in
// integer arithmetic ((n * l) mod N, as core.py:171 does before the float
// division), so a BandlimitedSignal source feeds the Hi-DFT without the host.

#include <algorithm>

#include "sfft_common.cuh"

namespace sfft {

constexpr int kSynthThreads = 256;
constexpr int kSynthTile = 1024;  // support elements staged in smem per round

__global__ void __launch_bounds__(kSynthThreads)
k_synthesize(const int64_t* __restrict__ J, const Cx<double>* __restrict__ c, int64_t k, int M,
             const int64_t* __restrict__ loc, int64_t n, Cx<double>* __restrict__ out) {
  __shared__ int64_t sJ[kSynthTile];
  __shared__ Cx<double> sc[kSynthTile];
  const uint64_t nmask = (1ull << M) - 1;
  const double inv_half_n = ldexp(1.0, 1 - M);  // 2/N: angle 2 pi m / N = pi * (2m/N)
  for (int64_t base = (int64_t)blockIdx.x * kSynthThreads; base < n; base += (int64_t)gridDim.x * kSynthThreads) {
    const int64_t i = base + threadIdx.x;
    const uint64_t li = i < n ? ((uint64_t)loc[i] & nmask) : 0;
    double ax = 0.0, ay = 0.0;
    for (int64_t j0 = 0; j0 < k; j0 += kSynthTile) {
      const int cnt = (int)std::min<int64_t>(kSynthTile, k - j0);
      __syncthreads();
      for (int e = threadIdx.x; e < cnt; e += kSynthThreads) {
        sJ[e] = J[j0 + e];
        sc[e] = c[j0 + e];
      }
      __syncthreads();
      for (int e = 0; e < cnt; ++e) {
        const uint64_t m = (li * (uint64_t)sJ[e]) & nmask;  // exact (n*l) mod N
        double sn, cs;
        sincospi((double)m * inv_half_n, &sn, &cs);
        ax = fma(sc[e].x, cs, fma(-sc[e].y, sn, ax));
        ay = fma(sc[e].x, sn, fma(sc[e].y, cs, ay));
      }
    }
    if (i < n) out[i] = Cx<double>{ax * ldexp(1.0, -M), ay * ldexp(1.0, -M)};
  }
}

}  // namespace sfft

using namespace sfft;

extern "C" int sfft_synthesize(const int64_t* J, const void* coeffs, int64_t k, int M, const int64_t* locations,
                               int64_t n, void* out, sfft_stream_t stream) {
  SFFT_NVTX("sfft_synthesize");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 62) return fail(SFFT_ERR_INVALID, "M out of range");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (n < 0) return fail(SFFT_ERR_INVALID, "negative location count");
  if (n == 0) return SFFT_OK;
  if (!J || !coeffs || !locations || !out) return fail(SFFT_ERR_INVALID, "null pointer");
  if (M > 31) return fail(SFFT_ERR_UNSUPPORTED, "synthesis needs (n*l) < 2^64: N <= 2^31");
  const int64_t blocks = std::min<int64_t>((n + kSynthThreads - 1) / kSynthThreads, (int64_t)num_sms() * 8);
  k_synthesize<<<(unsigned)blocks, kSynthThreads, 0, st>>>(J, (const Cx<double>*)coeffs, k, M, locations, n,
                                                           (Cx<double>*)out);
  SFFT_CUDA(cudaGetLastError());
  return SFFT_OK;
}

// ------------------------------------------------- FMA throughput probe ---
namespace sfft {

template <typename T, int CH>
__global__ void __launch_bounds__(256) k_fma_probe(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)12345) out[0] = s;  // never true: keeps the chains alive
}

template <typename T>
static int fma_probe(double* tflops, cudaStream_t st) {
  constexpr int CH = 8, NT = 256, ITERS = 4096;
  const int grid = num_sms() * 8;
  T* out = nullptr;
  SFFT_CUDA(cudaMalloc(&out, sizeof(T)));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  float best = 0.f;
  for (int rep = 0; rep < 4 && e == cudaSuccess; ++rep) {  // rep 0 warms up
    e = cudaEventRecord(e0, st);
    k_fma_probe<T, CH><<<grid, NT, 0, st>>>(out, rep == 0 ? 64 : ITERS, (T)0.999, (T)0.001);
    if (e == cudaSuccess) e = cudaEventRecord(e1, st);
    if (e == cudaSuccess) e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && e == cudaSuccess && (best == 0.f || ms < best)) best = ms;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(out);
  if (e != cudaSuccess) return cuda_fail(e, "FMA probe");
  *tflops = 2.0 * grid * NT * (double)ITERS * CH / (best * 1e-3) / 1e12;
  return SFFT_OK;
}

}  // namespace sfft

extern "C" int sfft_probe_fma_peak(int dtype, double* tflops, sfft_stream_t stream) {
  SFFT_NVTX("sfft_probe_fma_peak");
  if (!tflops) return sfft::fail(SFFT_ERR_INVALID, "sfft_probe_fma_peak: null output");
  if (dtype != SFFT_C64 && dtype != SFFT_C128) return sfft::fail(SFFT_ERR_INVALID, "sfft_probe_fma_peak: dtype");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return dtype == SFFT_C64 ? sfft::fma_probe<float>(tflops, st) : sfft::fma_probe<double>(tflops, st);
}
