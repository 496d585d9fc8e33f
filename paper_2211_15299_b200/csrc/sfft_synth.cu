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
