// Hi-DFT of a batch stored sample-major ("interleaved", an (N, B) matrix:
// sample n of signal b at signals[n * ld + b]).  In the row-major (B, N)
// layout every sample of configs 2-4 sits in its own 128 B line (the gather
// moves 16x its bytes); stored interleaved, the SG signals of a CTA read
// their sample n from one contiguous SG-element run, so the gather moves
// whole sectors of useful data.  Same plan, same butterfly and outputs as
// sfft_hidft (hidft.py:135-207): the batch layout is the only difference.
//
// Thread tid = g + SG * t: signal g of the CTA's group, thread t of the
// signal's butterfly (Geo<T,S>: E slots per thread).  A warp covers 32/SG
// slot positions of SG consecutive signals, so each gather instruction reads
// 32/SG contiguous runs of SG samples.  Each signal's slots live in its own
// shared-memory block, padded by 16 B so the SG blocks start on different
// banks.

#include "sfft_kernels.cuh"

namespace sfft {

template <typename T, int S, int SG>
struct NbGeo {
  using G = Geo<T, S>;
  static constexpr int TPS = G::TPS, NT = TPS * SG, PAD = 16 / (int)sizeof(Cx<T>);
  static constexpr int STRIDE = G::A + PAD;  // elements per signal block
  static constexpr size_t SMEM = (size_t)SG * STRIDE * sizeof(Cx<T>);
  static_assert(NT <= 1024, "interleaved kernel: SG thread groups per CTA");
};

template <typename T, int S, int SG>
__global__ void __launch_bounds__(NbGeo<T, S, SG>::NT) k_hidft_nb(const PlanArgs args) {
  using NG = NbGeo<T, S, SG>;
  using G = typename NG::G;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_release();
  const int tid = threadIdx.x;
  const int g = tid % SG, t = tid / SG;
  const int64_t b = (int64_t)blockIdx.x * SG + g;
  const bool live = b < args.B;
  const uint32_t nmask = (args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u);
  uint32_t d[S > 0 ? S : 1];
#pragma unroll
  for (int i = 0; i < S; ++i) d[i] = 1u << (args.M - 1 - args.used[i]);
  Cx<T> v[G::E];
  {
    const Cx<T>* col = reinterpret_cast<const Cx<T>*>(args.sig) + (live ? b : 0);
    uint32_t hi = args.negshift;
#pragma unroll
    for (int i = G::LE; i < S; ++i)
      if ((t >> (i - G::LE)) & 1) hi += d[i];
#pragma unroll
    for (int x = 0; x < G::E; ++x) {
      uint32_t off = hi;
#pragma unroll
      for (int i = 0; i < G::LE; ++i)
        if ((x >> i) & 1) off += d[i];
      v[x] = live ? load_sample(col + (int64_t)(off & nmask) * args.ld) : Cx<T>{T(0), T(0)};
    }
  }
  Cx<T>* sd = reinterpret_cast<Cx<T>*>(smem_raw) + g * NG::STRIDE;
  // the SG signals' butterflies share the CTA barrier of each pass
  butterfly<T, S>(v, t, sd, reinterpret_cast<const Cx<T>*>(args.tw));
  pdl_wait();  // earlier launches in the stream complete before the first store
  if (!live) return;
  const T scale = (T)args.scale1;
  Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + b * args.ld1;
  if (args.n1 == G::A && args.map1) {
    int a[G::E];
#pragma unroll
    for (int j = 0; j < G::E; ++j) a[j] = __ldg(args.map1 + t + j * G::TPS);
#pragma unroll
    for (int j = 0; j < G::E; ++j) o1[t + j * G::TPS] = cscale(sd[swz<T, S>(a[j])], scale);
  } else {
    for (int64_t i = t; i < args.n1; i += G::TPS) {
      const int a = args.map1 ? __ldg(args.map1 + i) : (int)i;
      o1[i] = cscale(sd[swz<T, S>(a)], scale);
    }
  }
}

#ifndef SFFT_NB_SG
#define SFFT_NB_SG 8
#endif

// signals per CTA: SFFT_NB_SG, fewer where the thread count (1024) or the
// shared memory (227 KB) of one CTA would not hold them
template <typename T, int S>
constexpr int nb_sg() {
  constexpr int tps = Geo<T, S>::TPS, a = 1 << S;
  int sg = SFFT_NB_SG;
  while (sg > 1 && (sg * tps > 1024 || (size_t)sg * (a + 2) * sizeof(Cx<T>) > 227 * 1024)) sg >>= 1;
  return sg;
}

template <typename T, int S>
static int run_nb(const PlanArgs& a, cudaStream_t st) {
  constexpr int SG = nb_sg<T, S>();
  using NG = NbGeo<T, S, SG>;
  auto kern = k_hidft_nb<T, S, SG>;
  int occ = 0;
  if (int rc = kernel_occupancy(kern, NG::NT, NG::SMEM, &occ)) return rc;
  const int64_t grid = (a.B + SG - 1) / SG;
  if (grid == 0) return SFFT_OK;
  // inputs: the whole (N, ld) matrix; outputs: B rows of n1
  const ByteRange in[1] = {{(uintptr_t)a.sig, (uintptr_t)a.sig + (size_t)((1ll << a.M) * a.ld) * sizeof(Cx<T>)}};
  const ByteRange outs[1] = {
      {(uintptr_t)a.out1, (uintptr_t)a.out1 + (size_t)((a.B - 1) * a.ld1 + a.n1) * sizeof(Cx<T>)}};
  const bool pdl = pdl_join(st, in, 1, outs, 1, true);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NG::NT);
  cfg.dynamicSmemBytes = NG::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  SFFT_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return SFFT_OK;
}

#define NB_CASE(S_, T_) case S_: return run_nb<T_, S_>(a, st);

static int dispatch_nb(const sfft_plan* p, const PlanArgs& a, cudaStream_t st) {
  if (p->dtype == SFFT_C64) {
    switch (p->s) {
      NB_CASE(1, float) NB_CASE(2, float) NB_CASE(3, float) NB_CASE(4, float) NB_CASE(5, float)
      NB_CASE(6, float) NB_CASE(7, float) NB_CASE(8, float) NB_CASE(9, float) NB_CASE(10, float)
      NB_CASE(11, float) NB_CASE(12, float)
      default: break;
    }
  } else {
    switch (p->s) {
      NB_CASE(1, double) NB_CASE(2, double) NB_CASE(3, double) NB_CASE(4, double) NB_CASE(5, double)
      NB_CASE(6, double) NB_CASE(7, double) NB_CASE(8, double) NB_CASE(9, double) NB_CASE(10, double)
      NB_CASE(11, double)
      default: break;
    }
  }
  return fail(SFFT_ERR_UNSUPPORTED, "interleaved layout: 2^s slots beyond 2^12 (c64) / 2^11 (c128)");
}

}  // namespace sfft

using namespace sfft;

extern "C" int sfft_hidft_interleaved(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
                                      int64_t shift, int out_kind, void* out, int64_t ld_out,
                                      sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_interleaved");
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(plan, "sfft_hidft_interleaved")) return rj;
  if (B < 0) return fail(SFFT_ERR_INVALID, "negative batch");
  if (B == 0) return SFFT_OK;
  if (!signals || !out) return fail(SFFT_ERR_INVALID, "null signal or output pointer");
  if (ld < B) return fail(SFFT_ERR_INVALID, "sample stride ld must be >= B");
  if (plan->s < 1) return fail(SFFT_ERR_UNSUPPORTED, "interleaved layout needs s >= 1");
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  if (dev != plan->device) return fail(SFFT_ERR_INVALID, "plan belongs to another device");
  const int32_t *map = nullptr, *inv = nullptr;
  int64_t n_out = 0;
  double scale = 1.0;
  if (int rc = out_spec(plan, out_kind, &map, &n_out, &scale, &inv)) return rc;
  if (ld_out < n_out) return fail(SFFT_ERR_INVALID, "output row stride too small");
  PlanArgs a{};
  a.sig = signals;
  a.B = B;
  a.ld = ld;
  a.M = plan->M;
  const int64_t N = 1ll << plan->M;
  const int64_t sh = ((shift % N) + N) % N;
  a.negshift = (uint32_t)((N - sh) & (N - 1));
  for (int i = 0; i < 32; ++i) a.used[i] = i < plan->s ? plan->used[i] : 0;
  a.tw = plan->d_twiddles;
  a.map1 = map;
  a.n1 = n_out;
  a.scale1 = scale;
  a.out1 = out;
  a.ld1 = ld_out;
  a.nshift = 1;
  return dispatch_nb(plan, a, (cudaStream_t)stream);
}
