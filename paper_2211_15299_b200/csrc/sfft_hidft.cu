// Hi-DFT transform kernels for sm_100a: gather -> generalised radix-2
// butterfly -> permuted, scaled store, one launch per batch.
//
// Reference: hidft.py:135-185 (hidft), hidft.py:188-207 (hidft_to_dft),
// sas.py:336-371 (sas_transform, mu*=1).
//
// Slot a (0 <= a < A = 2^s) holds, before stage 1, the sample at
//   off(a) = sum_i bit_i(a) 2^(M-1-used_i)            (hidft.py:155-158)
// and stage k pairs slots differing in bit k-1 with the twiddle
// tw_k[a mod 2^(k-1)]; branch 0 = v0 - w v1, branch 1 = v0 + w v1
// (hidft.py:160-167).  That is a radix-2 DIT network with data-dependent
// twiddles, so it is executed as a register-blocked Stockham-style FFT:
// every thread owns E slots, runs log2(E) stages in registers, and trades
// slots through (swizzled) shared memory between passes.
//
// Layout in HBM: signals are rows of N complex (c64 = float2, c128 =
// double2) with row stride ld; outputs are rows of n_out complex.

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sfft_kernels.cuh"

namespace sfft {

// One CTA per SPC signals, no per-CTA setup: the gather is the first thing
// every thread does, the butterfly reads the plan's twiddles through L1,
// and the block scheduler balances the grid over the 148 SMs.
#ifndef SFFT_PLAN_E14
#define SFFT_PLAN_E14 32
#endif
// slots per thread of the plan kernel (0: the type's default).  2^14-slot
// complex64 rows (config 3) use 32 per thread: 512 threads, three register
// passes (5 + 5 + 4 stages) instead of four, so the one CTA per SM spends
// less time in the butterfly with its share of HBM idle (209 -> 197 us)
// 2^13-slot complex128 rows: 16 per thread (512 threads, up to 128 registers)
// instead of 8 (1024 threads at 64 registers spilled 24 B)
template <typename T, int S> constexpr int plan_e() {
  return (sizeof(T) == 4 && S == 14) ? SFFT_PLAN_E14 : (sizeof(T) == 8 && S == 13) ? 16 : 0;
}

template <typename T, int S>
__global__ void __launch_bounds__(Geo<T, S, plan_e<T, S>()>::NT, Geo<T, S, plan_e<T, S>()>::MINB)
k_hidft_plan(const PlanArgs args) {
  constexpr int EO = plan_e<T, S>();
  using G = Geo<T, S, EO>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sdata = reinterpret_cast<Cx<T>*>(smem_raw);
  pdl_release();  // the next launch may start gathering (its inputs are checked on the host)
  const int tid = threadIdx.x;
  const int g = tid / G::TPS, t = tid % G::TPS;
  const int64_t b = (int64_t)blockIdx.x * G::SPC + g;  // output row
  const bool live = b < args.B * args.nshift;
  uint32_t d[S > 0 ? S : 1];
#pragma unroll
  for (int i = 0; i < S; ++i)
    d[i] = args.identity == 1   ? (1u << i)            // pre-gathered, slot order
           : args.identity == 2 ? (1u << (S - 1 - i))  // pre-gathered, sorted (pattern) order
                                : (1u << (args.M - 1 - args.used[i]));
  const uint32_t nmask = args.identity ? (uint32_t)(G::A - 1)
                                        : ((args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u));
  Cx<T> v[G::E];
  if (live) {
    // one row per signal (nshift == 1) skips the 64-bit division on the gather's critical path
    const int64_t bs = args.nshift == 1 ? b : b / args.nshift;
    const uint32_t rsh = args.nshift == 1 ? 0u : (uint32_t)(b % args.nshift);
    const uint32_t base = args.identity ? 0u : ((args.negshift - rsh) & nmask);
    if (sizeof(T) == 8 && args.in_c64)
      gather<T, S, float, EO>(v, t, reinterpret_cast<const Cx<float>*>(args.sig) + bs * args.ld, d, base, nmask);
    else
      gather<T, S, T, EO>(v, t, reinterpret_cast<const Cx<T>*>(args.sig) + bs * args.ld, d, base, nmask);
  } else {
#pragma unroll
    for (int x = 0; x < G::E; ++x) v[x] = Cx<T>{T(0), T(0)};
  }
  Cx<T>* sd = sdata + g * G::A;
  butterfly<T, S, false, EO>(v, t, sd, reinterpret_cast<const Cx<T>*>(args.tw));
  pdl_wait();  // earlier launches in the stream complete before the first store (see plan_pdl)
  if (live) {
    const T scale = (T)args.scale1;
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + b * args.ld1;
    if (args.n1 == G::A && args.map1) {  // one output per slot (homogeneous DFT order): unrolled, loads batched
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
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + b * args.ld2;
      for (int i = t; i < G::A; i += G::TPS) o2[i] = sd[swz<T, S>(i)];
    }
  }
}

// Programmatic dependent launch across calls (opt-in).  A kernel launched
// with the PDL attribute may start while its predecessor on the stream
// drains; the library's kernels read only their inputs (signals, supports,
// plan tables) before griddepcontrol.wait and store only after it.  That is
// safe when the predecessor is one of the library's own launches whose
// outputs the new launch does not read, but NOT when the predecessor is a
// foreign kernel that produced the inputs and triggered its dependents early
// (CUTLASS-style producers call launch_dependents before their last stores).
// The library cannot see foreign launches, so overlap across calls happens
// only inside a chain scope the caller opens on a stream
// (sfft_stream_chain(stream, 1): "consecutive library calls on this stream;
// no other kernel on it writes their inputs while the scope is open").  In a
// scope, launch N+1 joins the chain only if its inputs do not overlap any
// output of the chain since the last fully ordered launch (checked here),
// and the first launch after opening the scope is fully ordered.  Outside a
// scope (the default) the first kernel of every call is fully stream-ordered;
// kernels inside one call still chain among themselves.  SFFT_PDL=0
// disables PDL everywhere.
namespace {
struct PdlChain {
  bool scope = false;                                  // sfft_stream_chain(st, 1) in effect
  std::vector<std::pair<uintptr_t, uintptr_t>> outs;  // [lo, hi) written by the chain
};
std::mutex g_pdl_mu;
std::map<cudaStream_t, PdlChain> g_pdl;
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("SFFT_PDL");
    return !(e && atoi(e) == 0);
  }();
  return v;
}
}  // namespace

bool pdl_join(cudaStream_t st, const ByteRange* in, int nin, const ByteRange* out, int nout, bool eligible) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  PdlChain& c = g_pdl[st];
  // outside a scope the chain is always empty: the call's first launch is ordered
  bool ok = eligible && c.scope && pdl_enabled() && !c.outs.empty() && c.outs.size() < 16;
  for (const auto& o : c.outs)
    for (int i = 0; i < nin && ok; ++i)
      if (in[i].first < o.second && o.first < in[i].second) ok = false;
  if (!ok) c.outs.clear();  // fully ordered: the chain restarts here
  if (c.scope) {
    for (int i = 0; i < nout; ++i) {
      const ByteRange& o = out[i];
      if (o.first >= o.second) continue;
      bool seen = false;
      for (const auto& x : c.outs) seen |= (x == o);
      if (!seen) c.outs.push_back(o);
    }
  }
  return ok;
}

}  // namespace sfft

// Open (enable = 1) or close (0) a PDL chain scope on a stream (see pdl_join).
extern "C" int sfft_stream_chain(sfft_stream_t stream, int enable) {
  std::lock_guard<std::mutex> lk(sfft::g_pdl_mu);
  sfft::PdlChain& c = sfft::g_pdl[(cudaStream_t)stream];
  c.scope = enable != 0;
  c.outs.clear();  // the first launch after opening (or closing) is fully ordered
  return SFFT_OK;
}

namespace sfft {

template <typename T, int S>
static int run_plan_kernel(const PlanArgs& a, cudaStream_t st) {
  using G = Geo<T, S, plan_e<T, S>()>;
  constexpr size_t smem = plan_smem<T, S>();
  static_assert(smem <= 227 * 1024, "plan kernel smem");
  auto kern = k_hidft_plan<T, S>;
  int occ = 0;
  int rc = kernel_occupancy(kern, G::NT, smem, &occ);
  if (rc) return rc;
  const int64_t ngroups = (a.B * a.nshift + G::SPC - 1) / G::SPC;
  if (ngroups > 0x7fffffff) return fail(SFFT_ERR_UNSUPPORTED, "batch too large for one launch");
  if (ngroups == 0) return SFFT_OK;
  const size_t esz_in = (sizeof(T) == 8 && a.in_c64) ? 8 : sizeof(Cx<T>);
  const int64_t rows = a.B * a.nshift;
  const ByteRange in[1] = {{(uintptr_t)a.sig, (uintptr_t)a.sig + (size_t)((a.B - 1) * a.ld +
                                                    (a.identity ? G::A : (1ll << a.M))) * esz_in}};
  const ByteRange outs[2] = {
      {(uintptr_t)a.out1, (uintptr_t)a.out1 + (size_t)((rows - 1) * a.ld1 + a.n1) * sizeof(Cx<T>)},
      {(uintptr_t)a.out2, a.out2 ? (uintptr_t)a.out2 + (size_t)((rows - 1) * a.ld2 + G::A) * sizeof(Cx<T>) : 0}};
  const bool pdl = pdl_join(st, in, 1, outs, 2, a.identity == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ngroups);
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

int max_supported_s(int dtype) { return dtype == SFFT_C64 ? kMaxSplitS_c64 : kMaxSplitS_c128; }

#define SFFT_CASES_12(M_, ...) \
  M_(0, __VA_ARGS__) M_(1, __VA_ARGS__) M_(2, __VA_ARGS__) M_(3, __VA_ARGS__) M_(4, __VA_ARGS__) \
  M_(5, __VA_ARGS__) M_(6, __VA_ARGS__) M_(7, __VA_ARGS__) M_(8, __VA_ARGS__) M_(9, __VA_ARGS__) \
  M_(10, __VA_ARGS__) M_(11, __VA_ARGS__) M_(12, __VA_ARGS__)

#define PLAN_CASE(S_, T_) case S_: return run_plan_kernel<T_, S_>(a, st);

static int dispatch_plan(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  const int dtype = p->dtype, s = p->s;
  if (p->split_lc) return run_large(p, a, inv1, st);
  if (dtype == SFFT_C64) {
    switch (s) {
      SFFT_CASES_12(PLAN_CASE, float)
      PLAN_CASE(13, float)
      PLAN_CASE(14, float)
      default: break;
    }
  } else {
    switch (s) {
      SFFT_CASES_12(PLAN_CASE, double)
      PLAN_CASE(13, double)
      default: break;
    }
  }
  return fail(SFFT_ERR_UNSUPPORTED, "2^s slots exceed the single-CTA transform (s=" +
                                        std::to_string(s) + ")");
}

int launch_hidft_plan(const sfft_plan* p, const void* sig, int64_t B, int64_t ld, int64_t shift,
                      const int32_t* map1, const int32_t* inv1, int64_t n1, double scale1, void* out1,
                      int64_t ld1, void* out2, int64_t ld2, int identity, cudaStream_t st,
                      int64_t nshift, int in_c64) {
  PlanArgs a{};
  a.nshift = nshift > 0 ? nshift : 1;
  a.in_c64 = in_c64;
  a.identity = identity;
#ifdef SFFT_PHASE_TIMING
  if (const char* e = getenv("SFFT_DEBUG_SKIP")) a.debug_skip = atoi(e);
#endif
  a.sig = sig;
  a.B = B;
  a.ld = ld;
  a.M = p->M;
  const int64_t N = 1ll << p->M;
  const int64_t sh = ((shift % N) + N) % N;
  a.negshift = (uint32_t)((N - sh) & (N - 1));
  for (int i = 0; i < 32; ++i) a.used[i] = i < p->s ? p->used[i] : 0;
  a.tw = p->d_twiddles;
  a.map1 = map1;
  a.n1 = n1;
  a.scale1 = scale1;
  a.out1 = out1;
  a.ld1 = ld1;
  a.out2 = out2;
  a.ld2 = ld2;
  return dispatch_plan(p, a, inv1, st);
}

// 2^s beyond one CTA: the cluster kernel gathers in sorted order, so
// pre-gathered rows are best staged in that order (coalesced reads); the
// single-CTA kernel reads either order from L2-resident staging
bool gathered_sorted(const sfft_plan* p) {
  return p->s > (p->dtype == SFFT_C64 ? kMaxPlanS_c64 : kMaxPlanS_c128);
}

template <typename T>
__global__ void k_apply_map(const Cx<T>* __restrict__ in, int64_t B, int64_t ld_in,
                            const int32_t* __restrict__ map, int64_t n, T scale, Cx<T>* __restrict__ out,
                            int64_t ld_out) {
  const int64_t total = B * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / n, e = i % n;
    out[b * ld_out + e] = cscale(in[b * ld_in + map[e]], scale);
  }
}

// resolve (map, n_out, scale) for an output kind, checking its contract
int out_spec(const sfft_plan* plan, int out_kind, const int32_t** map, int64_t* n_out, double* scale,
             const int32_t** inv) {
  const double N = (double)(1ll << plan->M);
  *scale = 1.0;
  const int32_t* dummy;
  if (!inv) inv = &dummy;
  *inv = nullptr;
  switch (out_kind) {
    case SFFT_OUT_NODES:
      *inv = plan->d_inv_node;
      *map = plan->d_node_slots;
      *n_out = plan->n_nodes;
      return SFFT_OK;
    case SFFT_OUT_SLOTS:
      *map = nullptr;
      *n_out = plan->A;
      return SFFT_OK;
    case SFFT_OUT_DFT:  // hidft.py:196-207
      if (!plan->homogeneous)
        return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support");
      if (plan->height != 0)
        return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a height-0 transform");
      *map = plan->d_element_slots;
      *inv = plan->d_inv_elem;
      *n_out = plan->k;
      *scale = N / (double)plan->k;
      return SFFT_OK;
    case SFFT_OUT_SAS:  // sas.py:363-371, weight-1 nodes only
      if (plan->mu_star != 1)
        return fail(SFFT_ERR_CONTRACT, "mu* > 1: node systems need Vandermonde decoding");
      if (plan->height != 0) return fail(SFFT_ERR_CONTRACT, "sas decode needs height 0");
      *map = plan->d_element_slots;
      *inv = plan->d_inv_elem;
      *n_out = plan->k;
      *scale = N / (double)plan->A;
      return SFFT_OK;
    default:
      return fail(SFFT_ERR_INVALID, "unknown out_kind");
  }
}

}  // namespace sfft

// ------------------------------------------------------------------ C-ABI ---
using namespace sfft;

static int hidft_common(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
                        int64_t min_ld, int64_t shift, int out_kind, void* out, int64_t ld_out,
                        void* slot_out, int64_t ld_slot, int identity, cudaStream_t st) {
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (plan->per_signal) {  // sfft_plan_batched: supports derived on chip per signal
    if (identity) return reject_per_signal(plan, "sfft_hidft_gathered");
    if (out_kind != SFFT_OUT_DFT || shift != 0 || slot_out)
      return fail(SFFT_ERR_INVALID, "a per-signal plan serves SFFT_OUT_DFT at shift 0 without slot output");
    if (plan->n_supports != 1 && plan->n_supports != B)
      return fail(SFFT_ERR_INVALID, "batch size must equal the plan's number of supports");
    return fused_to_dft(plan->d_J, plan->k, plan->n_supports, plan->M, signals, B, ld, plan->dtype, out, ld_out,
                        nullptr, st);
  }
  if (B < 0) return fail(SFFT_ERR_INVALID, "negative batch");
  const int32_t* map = nullptr;
  const int32_t* inv = nullptr;
  int64_t n_out = 0;
  double scale = 1.0;
  int rc = out_spec(plan, out_kind, &map, &n_out, &scale, &inv);
  if (rc) return rc;
  if (B == 0) return SFFT_OK;
  if (!signals || !out) return fail(SFFT_ERR_INVALID, "null signal or output pointer");
  if (ld < min_ld) return fail(SFFT_ERR_INVALID, "signal row stride too small");
  if (ld_out < n_out) return fail(SFFT_ERR_INVALID, "output row stride too small");
  if (slot_out && ld_slot < plan->A) return fail(SFFT_ERR_INVALID, "slot row stride too small");
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  if (dev != plan->device) return fail(SFFT_ERR_INVALID, "plan belongs to another device");
  return launch_hidft_plan(plan, signals, B, ld, shift, map, inv, n_out, scale, out, ld_out, slot_out,
                           ld_slot, identity, st);
}

extern "C" int sfft_launch_count(const sfft_plan* plan, int64_t rows, int64_t* launches) {
  if (!plan || !launches) return fail(SFFT_ERR_INVALID, "null plan or output");
  if (rows < 0) return fail(SFFT_ERR_INVALID, "negative batch");
  *launches = rows > 0 ? 1 : 0;
  if (plan->per_signal || !plan->split_lc || rows == 0) return SFFT_OK;
  return large_launch_count(plan, rows, launches);
}

extern "C" int sfft_hidft(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
                          int64_t shift, int out_kind, void* out, int64_t ld_out, void* slot_out,
                          int64_t ld_slot, sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft");
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  return hidft_common(plan, signals, B, ld, 1ll << plan->M, shift, out_kind, out, ld_out, slot_out,
                      ld_slot, 0, (cudaStream_t)stream);
}

namespace sfft {
int hidft_gathered(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld, int sorted, int out_kind,
                   void* out, int64_t ld_out, void* slot_out, int64_t ld_slot, cudaStream_t st) {
  return hidft_common(plan, samples, B, ld, plan->A, 0, out_kind, out, ld_out, slot_out, ld_slot,
                      sorted ? 2 : 1, st);
}
}  // namespace sfft

extern "C" int sfft_hidft_staged(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld, int order,
                                 int out_kind, void* out, int64_t ld_out, void* slot_out, int64_t ld_slot,
                                 sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_staged");
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (order != SFFT_ORDER_SLOT && order != SFFT_ORDER_PATTERN) return fail(SFFT_ERR_INVALID, "unknown sample order");
  return hidft_gathered(plan, samples, B, ld, order == SFFT_ORDER_PATTERN, out_kind, out, ld_out, slot_out, ld_slot,
                        (cudaStream_t)stream);
}

extern "C" int sfft_hidft_gathered(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld,
                                   int out_kind, void* out, int64_t ld_out, void* slot_out,
                                   int64_t ld_slot, sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_gathered");
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  return hidft_common(plan, samples, B, ld, plan->A, 0, out_kind, out, ld_out, slot_out, ld_slot, 1,
                      (cudaStream_t)stream);
}

extern "C" int sfft_plan_apply_map(const sfft_plan* plan, int out_kind, const void* slot_values,
                                   int64_t B, int64_t ld, void* out, int64_t ld_out,
                                   sfft_stream_t stream) {
  SFFT_NVTX("sfft_plan_apply_map");
  cudaStream_t st = (cudaStream_t)stream;
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(plan, "sfft_plan_apply_map")) return rj;
  const int32_t* map = nullptr;
  int64_t n_out = 0;
  double scale = 1.0;
  int rc = out_spec(plan, out_kind, &map, &n_out, &scale);
  if (rc) return rc;
  if (!map) return fail(SFFT_ERR_INVALID, "slot output needs no map");
  if (B <= 0) return B < 0 ? fail(SFFT_ERR_INVALID, "negative batch") : SFFT_OK;
  if (ld < plan->A || ld_out < n_out) return fail(SFFT_ERR_INVALID, "row stride too small");
  const int64_t total = B * n_out;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
  if (plan->dtype == SFFT_C64)
    k_apply_map<float><<<grid, 256, 0, st>>>((const Cx<float>*)slot_values, B, ld, map, n_out,
                                             (float)scale, (Cx<float>*)out, ld_out);
  else
    k_apply_map<double><<<grid, 256, 0, st>>>((const Cx<double>*)slot_values, B, ld, map, n_out, scale,
                                              (Cx<double>*)out, ld_out);
  SFFT_CUDA(cudaGetLastError());
  return SFFT_OK;
}

namespace sfft {
int reject_per_signal(const sfft_plan* p, const char* entry) {
  if (p && p->per_signal)
    return fail(SFFT_ERR_INVALID, std::string(entry) + ": a per-signal plan (sfft_plan_batched) only serves "
                                                       "sfft_hidft with SFFT_OUT_DFT");
  return SFFT_OK;
}
}  // namespace sfft
