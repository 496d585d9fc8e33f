// Fused hidft + hidft_to_dft for homogeneous supports (config 4 per-signal
// supports, and shared supports without a host plan): pivots, pattern and
// twiddles are derived on chip per CTA, so one launch does plan + gather +
// butterfly + scaled, ascending-J store.
//
// Reference: congruence.py:76-101 (pivots), hidft.py:53-95 (_build_plan),
// hidft.py:135-207 (hidft, hidft_to_dft).

#include <algorithm>
#include <string>
#include <vector>

#include "sfft_kernels.cuh"

namespace sfft {

// -------------------------------------------- fused homogeneous to_dft ---
//
// pivots(J) for a homogeneous J without sorting: every pivot shows up as
// v2(j - j0) for the fixed element j0 (all nodes at a pivot level split), so
// P0 = OR_e 1 << ctz(j_e ^ j_0).  J is homogeneous iff |J| = 2^|P0|, the
// pattern map j -> pext(j, P0) is a bijection onto [0, 2^s), and for every
// slot x != 0 the element at x and the one at x minus its top bit first
// differ exactly at the pivot of that top bit (then every pairwise v2 lies in
// P0; congruence.py:235-241).  Representatives of every slot prefix are the
// elements at slot h < 2^(k-1) (all members of a prefix agree below the next
// pivot), which gives the twiddles of hidft.py:81-83.

struct FusedArgs {
  const int64_t* J;  // n_supports x k
  int64_t n_supports;
  const void* sig;
  int64_t B, ld;
  int M;
  void* out;
  int64_t ld_out;
  int32_t* status;  // n_supports
  int identity;     // rows pre-gathered in each row's own slot order (ld >= A)
};

// Plan for one support on `nthr` threads (tid in [0, nthr)).  Every thread
// of the CTA must call it at the same time (it uses CTA barriers); several
// thread groups may build several plans concurrently.  Writes spats
// (element -> slot), stw (A-1 twiddles) and the pivots (sctl + 2).
// scratch: 2*A ints.  Returns 0 ok, 2 invalid support, 3 not homogeneous.
template <typename T, int S>
__device__ int fused_plan(const int64_t* __restrict__ Jrow, bool live, int M, int tid, int nthr,
                          int* spats, Cx<T>* stw, int* scratch, int* sctl) {
  using G = Geo<T, S>;
  constexpr int A = G::A;
  int* sJ = scratch;
  int* sElem = scratch + A;
  int* spiv = sctl + 2;  // sctl[0] = pivot mask P0, sctl[1] = status
  const int64_t N = 1ll << M;
  if (tid == 0) { sctl[0] = 0; sctl[1] = 0; }
  __syncthreads();
  int bad = 0;
  if (live) {
    for (int e = tid; e < A; e += nthr) {
      const int64_t j = Jrow[e];
      if (j < 0 || j >= N) bad = 2;
      sJ[e] = (int)(j & (N - 1));
    }
  }
  __syncthreads();
  uint32_t mask = 0;
  if (live) {
    const int j0 = sJ[0];
    for (int e = tid; e < A; e += nthr) {
      const int j = sJ[e];
      if (e > 0) {
        if (sJ[e - 1] >= j) bad = 2;
        else mask |= 1u << (__ffs(j ^ j0) - 1);
      }
    }
  }
  if (mask) atomicOr(reinterpret_cast<unsigned*>(&sctl[0]), mask);
  if (bad) atomicMax(&sctl[1], bad);
  __syncthreads();
  mask = (uint32_t)sctl[0];
  const bool go = live && sctl[1] == 0 && __popc(mask) == S;
  if (go)
    for (int i = tid; i < S; i += nthr) spiv[i] = (int)__fns(mask, 0, i + 1);
  __syncthreads();
  int piv[S > 0 ? S : 1];
  if (go) {
#pragma unroll
    for (int i = 0; i < S; ++i) piv[i] = spiv[i];
    for (int e = tid; e < A; e += nthr) {
      const uint32_t j = (uint32_t)sJ[e];
      uint32_t p = 0;
#pragma unroll
      for (int i = 0; i < S; ++i) p |= ((j >> piv[i]) & 1u) << i;
      spats[e] = (int)p;
      sElem[p] = (int)j;
    }
  }
  __syncthreads();
  if (go) {
    bad = 0;
    for (int e = tid; e < A; e += nthr)
      if (sElem[spats[e]] != sJ[e]) bad = 3;  // two elements share a pattern
    for (int x = tid + 1; x < A; x += nthr) {
      const int top = 31 - __clz(x);
      const uint32_t dd = (uint32_t)(sElem[x] ^ sElem[x ^ (1 << top)]);
      if (dd == 0 || __ffs(dd) - 1 != spiv[top]) bad = 3;  // v2 outside P0
    }
    if (bad) atomicMax(&sctl[1], bad);
    for (int idx = tid; idx < A - 1; idx += nthr) {
      const int beta = 31 - __clz(idx + 1);
      const int h = idx + 1 - (1 << beta);
      const int rk = spiv[beta];
      const uint32_t shared = (uint32_t)sElem[h] & ((1u << rk) - 1u);
      stw[idx] = twiddle<T>(shared, rk);
    }
  }
  __syncthreads();
  if (!live) return 0;
  if (sctl[1] != 0) return sctl[1];
  return __popc(mask) == S ? 0 : 3;
}

// Slots per thread of the fused kernel: with per-signal plans (config 4) the
// on-chip plan derivation is spread over the signal's threads, so complex64
// uses 8 slots per thread (twice the threads of the plan kernel's 16):
// config 4 221 -> 198 us.  The shared-support variant keeps the default.
#ifndef SFFT_FUSED_E
#define SFFT_FUSED_E 8
#endif
template <typename T, int S, bool PS>
constexpr int fused_e() { return (PS && sizeof(T) == 4 && S >= 7) ? SFFT_FUSED_E : 0; }

template <typename T, int S, bool PS> constexpr size_t fused_smem() {
  using G = Geo<T, S, fused_e<T, S, PS>()>;
  constexpr size_t NP = PS ? G::SPC : 1;
  return (size_t)G::SPC * G::A * sizeof(Cx<T>) + NP * (G::A > 1 ? G::A - 1 : 1) * sizeof(Cx<T>) +
         NP * G::A * sizeof(int);
}

// PER_SIGNAL: one CTA per SPC signals, each group derives its own support's
// plan on chip, then gathers, transforms and stores.  Shared support: CTAs
// are persistent, build the one plan once and loop over signal groups.
template <typename T, int S, bool PER_SIGNAL>
__global__ void __launch_bounds__(Geo<T, S, fused_e<T, S, PER_SIGNAL>()>::NT,
                                  Geo<T, S, fused_e<T, S, PER_SIGNAL>()>::MINB)
k_fused_to_dft(const FusedArgs args) {
  constexpr int EO = fused_e<T, S, PER_SIGNAL>();
  using G = Geo<T, S, EO>;
  constexpr int A = G::A;
  constexpr int NP = PER_SIGNAL ? G::SPC : 1;  // plans held per CTA
  constexpr int TWN = A > 1 ? A - 1 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sdata = reinterpret_cast<Cx<T>*>(smem_raw);            // SPC * A
  Cx<T>* stw_all = sdata + G::SPC * A;                          // NP * TWN
  int* spats_all = reinterpret_cast<int*>(stw_all + NP * TWN);  // NP * A
  __shared__ int sctl[NP][2 + (S > 0 ? S : 1)];

  if (PER_SIGNAL) pdl_release();  // the next launch may start gathering (inputs checked on the host)
  const int tid = threadIdx.x;
  const int g = tid / G::TPS, t = tid % G::TPS;
  const uint32_t nmask = (args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u);
  const T scale = (T)((double)(1ll << args.M) / (double)A);
  Cx<T>* sd = sdata + g * A;
  const int pg = PER_SIGNAL ? g : 0;
  int* pats = spats_all + pg * A;
  Cx<T>* tw = stw_all + pg * TWN;
  const int* spiv = &sctl[pg][2];

  int64_t grp = blockIdx.x, step = gridDim.x;
  const int64_t ngroups = (args.B + G::SPC - 1) / G::SPC;
  if (!PER_SIGNAL) {
    // one plan per CTA, built by all its threads; scratch aliases the data area
    const int st = fused_plan<T, S>(args.J, true, args.M, tid, G::NT, pats, tw,
                                    reinterpret_cast<int*>(sdata), &sctl[0][0]);
    if (blockIdx.x == 0 && tid == 0 && args.status) args.status[0] = st;
    if (st != 0) return;  // uniform across the CTA
  }
  for (; grp < ngroups; grp += step) {
    const int64_t b = grp * G::SPC + g;
    const bool live = b < args.B;
    int st = 0;
    if (PER_SIGNAL) {
      st = fused_plan<T, S>(args.J + (live ? b : 0) * (int64_t)A, live, args.M, t, G::TPS, pats, tw,
                            reinterpret_cast<int*>(sd), &sctl[g][0]);
    }
    const bool ok = live && st == 0;
    Cx<T> v[G::E];
    if (ok) {
      uint32_t d[S > 0 ? S : 1];
#pragma unroll
      for (int i = 0; i < S; ++i) d[i] = args.identity ? (1u << i) : (1u << (args.M - 1 - spiv[i]));
      const Cx<T>* row = reinterpret_cast<const Cx<T>*>(args.sig) + b * args.ld;
      gather<T, S, T, EO>(v, t, row, d, 0u, args.identity ? (uint32_t)(A - 1) : nmask);
    } else {
#pragma unroll
      for (int x = 0; x < G::E; ++x) v[x] = Cx<T>{T(0), T(0)};
    }
    butterfly<T, S, false, EO>(v, t, sd, tw);
    if (PER_SIGNAL) {
      pdl_wait();  // earlier launches complete before the first store
      if (live && t == 0 && args.status) args.status[b] = st;
    }
    if (ok) {
      Cx<T>* o = reinterpret_cast<Cx<T>*>(args.out) + b * args.ld_out;
      for (int i = t; i < A; i += G::TPS) o[i] = cscale(sd[swz<T, S>(pats[i])], scale);
    }
    __syncthreads();
  }
}

template <typename T, int S, bool PS>
static int run_fused_kernel(const FusedArgs& a, cudaStream_t st, bool pdl_ok) {
  using G = Geo<T, S, fused_e<T, S, PS>()>;
  constexpr size_t smem = fused_smem<T, S, PS>();
  static_assert(smem <= 227 * 1024, "fused kernel smem");
  auto kern = k_fused_to_dft<T, S, PS>;
  int occ = 0;
  int rc = kernel_occupancy(kern, G::NT, smem, &occ);
  if (rc) return rc;
  const int64_t ngroups = (a.B + G::SPC - 1) / G::SPC;
  int64_t grid = PS ? ngroups : std::min<int64_t>(ngroups, (int64_t)num_sms() * occ);
  if (grid > 0x7fffffff) return fail(SFFT_ERR_UNSUPPORTED, "batch too large for one launch");
  // per-signal plans join the stream's PDL chain like the plan kernel
  // (sfft_hidft.cu, pdl_join): signals and supports are read before the wait
  constexpr size_t esz = sizeof(Cx<T>);
  const ByteRange in[2] = {
      {(uintptr_t)a.sig, (uintptr_t)a.sig + (size_t)((a.B - 1) * a.ld + (a.identity ? G::A : (1ll << a.M))) * esz},
      {(uintptr_t)a.J, (uintptr_t)a.J + (size_t)a.n_supports * G::A * sizeof(int64_t)}};
  const ByteRange outs[2] = {
      {(uintptr_t)a.out, (uintptr_t)a.out + (size_t)((a.B - 1) * a.ld_out + G::A) * esz},
      {(uintptr_t)a.status, a.status ? (uintptr_t)(a.status + a.n_supports) : 0}};
  const bool pdl = pdl_join(st, in, 2, outs, 2, PS && pdl_ok && !a.identity);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::max<int64_t>(grid, 1));
  cfg.blockDim = dim3(G::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  SFFT_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return SFFT_OK;
}

#define SFFT_CASES_12(M_, ...) \
  M_(0, __VA_ARGS__) M_(1, __VA_ARGS__) M_(2, __VA_ARGS__) M_(3, __VA_ARGS__) M_(4, __VA_ARGS__) \
  M_(5, __VA_ARGS__) M_(6, __VA_ARGS__) M_(7, __VA_ARGS__) M_(8, __VA_ARGS__) M_(9, __VA_ARGS__) \
  M_(10, __VA_ARGS__) M_(11, __VA_ARGS__) M_(12, __VA_ARGS__)
#define FUSED_CASE(S_, T_, PS_) case S_: return run_fused_kernel<T_, S_, PS_>(a, st, pdl_ok);

template <bool PS>
static int dispatch_fused(int dtype, int s, const FusedArgs& a, cudaStream_t st, bool pdl_ok) {
  if (dtype == SFFT_C64) {
    switch (s) {
      SFFT_CASES_12(FUSED_CASE, float, PS)
      FUSED_CASE(13, float, PS)
      default: break;
    }
  } else {
    switch (s) {
      SFFT_CASES_12(FUSED_CASE, double, PS)
      default: break;
    }
  }
  return fail(SFFT_ERR_UNSUPPORTED, "2^s slots exceed the fused single-CTA transform (s=" +
                                        std::to_string(s) + ")");
}

}  // namespace sfft

using namespace sfft;

extern "C" int sfft_hidft_to_dft_fused(const int64_t* J, int64_t k, int64_t n_supports, int M,
                                       const void* signals, int64_t B, int64_t ld, int dtype,
                                       void* out, int64_t ld_out, int32_t* status,
                                       sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_to_dft_fused");
  return fused_to_dft(J, k, n_supports, M, signals, B, ld, dtype, out, ld_out, status, (cudaStream_t)stream);
}

int sfft::fused_to_dft(const int64_t* J, int64_t k, int64_t n_supports, int M, const void* signals, int64_t B,
                       int64_t ld, int dtype, void* out, int64_t ld_out, int32_t* status, cudaStream_t st,
                       int identity) {
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (dtype != SFFT_C64 && dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown dtype");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (B < 0 || (n_supports != 1 && n_supports != B))
    return fail(SFFT_ERR_INVALID, "n_supports must be 1 or B");
  if (B == 0) return SFFT_OK;
  if (!J || !signals || !out) return fail(SFFT_ERR_INVALID, "null pointer");
  if (ld < (identity ? k : (1ll << M))) return fail(SFFT_ERR_INVALID, "signal row stride too small");
  if (ld_out < k) return fail(SFFT_ERR_INVALID, "output row stride too small");
  if (k & (k - 1)) return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support");
  const int s = 63 - __builtin_clzll((unsigned long long)k);
  if (s > (dtype == SFFT_C64 ? kMaxFusedS_c64 : kMaxFusedS_c128))
    return fail(SFFT_ERR_UNSUPPORTED, "fused transform limited to 2^" +
                                          std::to_string(dtype == SFFT_C64 ? kMaxFusedS_c64
                                                                           : kMaxFusedS_c128) +
                                          " slots");
  const int64_t* dJ = J;
  int64_t* tmpJ = nullptr;
  if (!is_device_pointer(J)) {
    SFFT_CUDA(cudaMallocAsync((void**)&tmpJ, sizeof(int64_t) * k * n_supports, st));
    SFFT_CUDA(cudaMemcpyAsync(tmpJ, J, sizeof(int64_t) * k * n_supports, cudaMemcpyHostToDevice, st));
    dJ = tmpJ;
  }
  int32_t* dstat = status;
  int32_t* tmpStat = nullptr;
  if (!dstat) {
    SFFT_CUDA(cudaMallocAsync((void**)&tmpStat, sizeof(int32_t) * n_supports, st));
    SFFT_CUDA(cudaMemsetAsync(tmpStat, 0, sizeof(int32_t) * n_supports, st));
    dstat = tmpStat;
  }
  FusedArgs a{};
  a.J = dJ;
  a.n_supports = n_supports;
  a.sig = signals;
  a.B = B;
  a.ld = ld;
  a.M = M;
  a.out = out;
  a.ld_out = ld_out;
  a.status = dstat;
  a.identity = identity;
  // no PDL after this call's own staging copies / memsets (only kernel-to-kernel overlap)
  const bool pdl_ok = !tmpJ && !tmpStat;
  int rc = (n_supports == 1 && B >= 1) ? dispatch_fused<false>(dtype, s, a, st, pdl_ok)
                                       : dispatch_fused<true>(dtype, s, a, st, pdl_ok);
  if (rc == SFFT_OK && tmpStat) {
    std::vector<int32_t> h(n_supports);
    cudaError_t e = cudaMemcpyAsync(h.data(), tmpStat, sizeof(int32_t) * n_supports,
                                    cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "status readback");
    for (int64_t i = 0; rc == SFFT_OK && i < n_supports; ++i) {
      if (h[i] == 2) rc = fail(SFFT_ERR_INVALID, "support " + std::to_string(i) + " is not a valid SupportSet");
      else if (h[i] == 3) rc = fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support (support " + std::to_string(i) + ")");
    }
  }
  if (tmpJ) cudaFreeAsync(tmpJ, st);
  if (tmpStat) cudaFreeAsync(tmpStat, st);
  return rc;
}
