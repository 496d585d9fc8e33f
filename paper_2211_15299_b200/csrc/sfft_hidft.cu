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

#include <cooperative_groups.h>

#include "sfft_common.cuh"
#include "sfft_plan.h"

namespace cg = cooperative_groups;

namespace sfft {

constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

template <typename T> struct EMax;
template <> struct EMax<float> { static constexpr int v = 16; static constexpr int SWZ = 4; };
template <> struct EMax<double> { static constexpr int v = 8; static constexpr int SWZ = 3; };

template <typename T, int S, int EOV = 0>
struct Geo {
  static constexpr int A = 1 << S;
  static constexpr int EM = EOV ? EOV : EMax<T>::v;
  static constexpr int E = A < EM ? A : EM;                   // slots per thread
  static constexpr int LE = ilog2c(E);
  static constexpr int TPS = A / E;                           // threads per signal
  static constexpr int NT = TPS > 64 ? TPS : 64;              // threads per CTA
  static constexpr int SPC = NT / TPS;                        // signals per CTA
  static constexpr int NPASS = S == 0 ? 1 : (S + LE - 1) / LE;
  // occupancy hint: >= 16 resident warps per SM where the register file allows
  static constexpr int MINB = NT >= 1024 ? 1 : (512 / NT > 1 ? 512 / NT : 1);
};

// Bank-conflict-free shared-memory slot position: XOR the low SWZ bits with
// the XOR-fold of the higher bits.  A bijection inside each aligned block,
// conflict-free for every power-of-two lane stride used below, and LINEAR
// over GF(2): swz(a ^ b) = swz(a) ^ swz(b), so a slot split into a thread
// part and a register part costs one XOR per access (the register part is
// a compile-time constant after unrolling).
template <typename T, int S>
__host__ __device__ constexpr int swz(int a) {
  constexpr int B = EMax<T>::SWZ;
  int y = a >> B, f = 0;
  for (int i = 0; i < (S + B - 1) / B; ++i) {
    f ^= y & ((1 << B) - 1);
    y >>= B;
  }
  return a ^ f;
}

// Slot owned by thread t (within its signal) for register x in pass p:
// bits [w0, w0+LE) come from x, the rest from t.
__host__ __device__ constexpr int pass_w0(int p, int S, int LE) { return (p * LE < S - LE) ? p * LE : S - LE; }
template <int S, int LE>
__device__ __forceinline__ int slot_t(int p, int t) {
  const int w0 = pass_w0(p, S, LE);
  return (t & ((1 << w0) - 1)) | ((t >> w0) << (w0 + LE));
}
template <int S, int LE>
__host__ __device__ constexpr int slot_x(int p, int x) { return x << pass_w0(p, S, LE); }
template <int S, int LE>
__device__ __forceinline__ int slot_of(int p, int t, int x) { return slot_t<S, LE>(p, t) | slot_x<S, LE>(p, x); }

// Stages [p*LE, min(p*LE+LE, S)) of pass p, in registers.
template <typename T, int S, int E, int LE>
__device__ __forceinline__ void pass_stages(Cx<T> (&v)[E], int p, int t, const Cx<T>* __restrict__ tw) {
  const int b0 = p * LE;
  const int b1 = (b0 + LE < S) ? b0 + LE : S;
  const int w0 = (b0 < S - LE) ? b0 : S - LE;
#pragma unroll
  for (int beta = b0; beta < b1; ++beta) {
    const int lb = beta - w0;
#pragma unroll
    for (int x = 0; x < E; ++x) {
      if (x & (1 << lb)) continue;
      const int a = slot_of<S, LE>(p, t, x);
      const int h = a & ((1 << beta) - 1);
      bfly(v[x], v[x | (1 << lb)], tw[(1 << beta) - 1 + h]);
    }
  }
}

// Whole butterfly for one signal per thread group.  On entry v holds the
// pass-0 slots (x + t*E) unless LOAD0 (then they are read from sd); on exit
// the slot values sit in sd (swizzled) and the CTA has passed a barrier.
template <typename T, int S, bool LOAD0 = false, int EOV = 0>
__device__ __forceinline__ void butterfly(Cx<T> (&v)[Geo<T, S, EOV>::E], int t, Cx<T>* sd,
                                          const Cx<T>* __restrict__ tw) {
  using G = Geo<T, S, EOV>;
#pragma unroll
  for (int p = 0; p < G::NPASS; ++p) {
    const int tb = swz<T, S>(slot_t<S, G::LE>(p, t));
    if (p > 0 || LOAD0) {
#pragma unroll
      for (int x = 0; x < G::E; ++x) v[x] = sd[tb ^ swz<T, S>(slot_x<S, G::LE>(p, x))];
    }
    pass_stages<T, S, G::E, G::LE>(v, p, t, tw);
#pragma unroll
    for (int x = 0; x < G::E; ++x) sd[tb ^ swz<T, S>(slot_x<S, G::LE>(p, x))] = v[x];
    __syncthreads();
  }
}

// Pass-0 gather: slot a = x + t*E reads sample (off(a) + base) mod N with
// off(a) = sum_i bit_i(a) d_i, d_i = 2^(M-1-used_i) (hidft.py:155-158).  The
// low LE bits of a come from the unrolled register index x, so their part
// of the offset is a compile-time selection of d_0..d_{LE-1}.  All E loads
// are issued back to back before any use.
template <typename T, int S, typename In = T>
__device__ __forceinline__ void gather(Cx<T> (&v)[Geo<T, S>::E], int t, const Cx<In>* __restrict__ row,
                                       const uint32_t (&d)[S > 0 ? S : 1], uint32_t base, uint32_t nmask) {
  using G = Geo<T, S>;
  uint32_t hi = base;
#pragma unroll
  for (int i = G::LE; i < S; ++i)
    if ((t >> (i - G::LE)) & 1) hi += d[i];
#pragma unroll
  for (int x = 0; x < G::E; ++x) {
    uint32_t off = hi;
#pragma unroll
    for (int i = 0; i < G::LE; ++i)
      if ((x >> i) & 1) off += d[i];
    const Cx<In> s = load_sample(row + (off & nmask));
    v[x] = Cx<T>{(T)s.x, (T)s.y};  // complex64 input into the fp64 path promotes exactly
  }
}

// ------------------------------------------------------ plan-driven kernel ---

struct PlanArgs {
  const void* sig;
  int64_t B, ld;
  int M;
  uint32_t negshift;
  int32_t used[32];
  const void* tw;       // A-1 twiddles in HBM, read through L1 (shared by all CTAs of an SM)
  const int32_t* map1;  // NULL => identity
  int64_t n1;
  double scale1;
  void* out1;
  int64_t ld1;
  void* out2;  // optional slot values (identity map)
  int64_t ld2;
  int identity;  // samples already gathered in slot order (row[a] = slot a)
  int in_c64;    // fp64 plan reading complex64 signals (promoted on load, as hidft.py:46 does)
  int64_t nshift;  // rows per signal: row r transforms signal r / nshift at shift shift0 + r % nshift
  int debug_skip;  // timing build only: bit0 gather, bit1 scatter, bit2 local stages, bit3 phase 2
};

template <typename T, int S> constexpr size_t plan_smem() {
  return (size_t)Geo<T, S>::SPC * Geo<T, S>::A * sizeof(Cx<T>);
}

// One CTA per SPC signals, no per-CTA setup: the gather is the first thing
// every thread does, the butterfly reads the plan's twiddles through L1,
// and the block scheduler balances the grid over the 148 SMs.
template <typename T, int S>
__global__ void __launch_bounds__(Geo<T, S>::NT, Geo<T, S>::MINB)
k_hidft_plan(const PlanArgs args) {
  using G = Geo<T, S>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sdata = reinterpret_cast<Cx<T>*>(smem_raw);
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
    const int64_t bs = b / args.nshift;
    const uint32_t base = args.identity ? 0u : ((args.negshift - (uint32_t)(b % args.nshift)) & nmask);
    if (sizeof(T) == 8 && args.in_c64)
      gather<T, S, float>(v, t, reinterpret_cast<const Cx<float>*>(args.sig) + bs * args.ld, d, base, nmask);
    else
      gather<T, S>(v, t, reinterpret_cast<const Cx<T>*>(args.sig) + bs * args.ld, d, base, nmask);
  } else {
#pragma unroll
    for (int x = 0; x < G::E; ++x) v[x] = Cx<T>{T(0), T(0)};
  }
  Cx<T>* sd = sdata + g * G::A;
  butterfly<T, S>(v, t, sd, reinterpret_cast<const Cx<T>*>(args.tw));
  if (live) {
    const T scale = (T)args.scale1;
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + b * args.ld1;
    for (int64_t i = t; i < args.n1; i += G::TPS) {
      const int a = args.map1 ? __ldg(args.map1 + i) : (int)i;
      o1[i] = cscale(sd[swz<T, S>(a)], scale);
    }
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + b * args.ld2;
      for (int i = t; i < G::A; i += G::TPS) o2[i] = sd[swz<T, S>(i)];
    }
  }
}

// ------------------------------------------ cluster kernel for large A ---
//
// 2^s slots beyond one SM's shared memory (config 5: A = 65536) are spread
// over a thread-block cluster of C CTAs; CTA q owns the slots whose top
// log2(C) bits equal q (so stages 1..s-log2(C) are CTA-local).
//  0. gather: CTA q loads the q-th contiguous chunk of the SORTED sample set
//     I_r (coalesced whenever the pattern has contiguous runs), and stores
//     each sample straight into its owner CTA's shared memory over DSMEM
//     (sorted index qs holds slot brev_s(qs)).
//  1. every CTA runs the local stages on its slice (the single-CTA code).
//  2. the last log2(C) stages: each CTA takes 1/C of the local indices,
//     reads the C partners of each from the C slices over DSMEM, finishes
//     the butterfly in registers and stores straight to the output row
//     through the plan's slot -> output-position map.
template <int S>
__device__ __forceinline__ uint32_t brev_s(uint32_t x) { return __brev(x) >> (32 - S); }

// --- DSMEM helpers (PTX): shared::cluster addresses, async remote stores that
// complete on the destination CTA's mbarrier, and the cluster barrier halves.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(uint32_t addr, Cx<float> v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               :: "r"(addr), "f"(v.x), "f"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async(uint32_t addr, Cx<double> v, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(addr), "d"(v.x), "d"(v.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(mbar), "r"(parity) : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive_tx_local(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

#ifdef SFFT_PHASE_TIMING
#define SFFT_SKIP(bit) (args.debug_skip & (1 << (bit)))
#else
#define SFFT_SKIP(bit) 0
#endif
#ifdef SFFT_PHASE_TIMING
// debug build only: per-CTA clock64 stamps at phase boundaries
__device__ unsigned long long g_phase_stamps[1 << 20][8];
#define SFFT_STAMP(i)                                                               \
  do {                                                                              \
    if (threadIdx.x == 0 && blockIdx.x < (1u << 20)) g_phase_stamps[blockIdx.x][i] = clock64(); \
  } while (0)
// accumulate time since the previous mark into slot i (thread 0)
#define SFFT_ACC_INIT() unsigned long long acc_t0__ = clock64()
#define SFFT_ACC(i)                                                                   \
  do {                                                                                \
    if (threadIdx.x == 0 && blockIdx.x < (1u << 20)) {                               \
      const unsigned long long t__ = clock64();                                        \
      g_phase_stamps[blockIdx.x][i] += t__ - acc_t0__;                                 \
      acc_t0__ = t__;                                                                  \
    }                                                                                 \
  } while (0)
#else
#define SFFT_STAMP(i) do {} while (0)
#define SFFT_ACC_INIT() do {} while (0)
#define SFFT_ACC(i) do {} while (0)
#endif

// 16-byte remote async store into another CTA's shared memory, completing on
// that CTA's mbarrier (two complex64 or one complex128)
__device__ __forceinline__ void st_async16(uint32_t addr, Cx<float> a, Cx<float> b, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(addr), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "r"(mbar) : "memory");
}
__device__ __forceinline__ void st_async16(uint32_t addr, Cx<double> a, Cx<double>, uint32_t mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               :: "r"(addr), "d"(a.x), "d"(a.y), "r"(mbar) : "memory");
}

template <typename T> struct ClusterE { static constexpr int v = 16; };  // slots per thread in the cluster kernel (8 measured 23% slower)
template <> struct ClusterE<double> { static constexpr int v = 8; };

template <typename T, int S, int C>
struct ClusterGeo {
  static constexpr int LC = ilog2c(C), SL = S - LC, AL = 1 << SL, PER = AL / C;
  static constexpr int EC = ClusterE<T>::v;
  using G = Geo<T, SL, EC>;
  static constexpr int NT = G::NT;
  static constexpr int EPU = 16 / (int)sizeof(Cx<T>);  // elements per 16-byte unit
  static constexpr size_t SMEM = 3 * (size_t)AL * sizeof(Cx<T>);  // W, R1, R2
  static constexpr int MINB = (int)((200 * 1024) / SMEM) >= 2 ? 2 : 1;
};

// Persistent cluster kernel (C CTAs per signal, clusters loop over signals).
// Per signal, two all-to-all exchanges of contiguous 16-byte blocks pushed
// with st.async into the receiver's buffer and counted by its mbarrier; no
// cluster-wide barrier inside the loop (a sender can only run ahead into
// the next signal after the receiver has released the buffer, see below).
//   0. CTA q gathers the q-th contiguous chunk of the SORTED sample set
//      (coalesced over runs; prefetched during the previous signal), stages
//      it in W grouped by owner CTA, and pushes block r to CTA r's R1
//      (layout [source q][i]).
//   1. CTA r transforms its slice (slots with top log2(C) bits = r, the
//      local stages 1..SL) reading pass 0 straight from R1, result in W.
//   2. CTA r pushes local slot range [q'*PER, (q'+1)*PER) to CTA q''s R2.
//   3. CTA q' finishes stages SL+1..S for its PER local indices (all C
//      partners in R2) and stores through the slot -> output map.
// Buffer reuse: R1 of signal n+1 is written by a sender only after that
// sender finished step 3 of signal n, which needed this CTA's step-2 data,
// which this CTA sends after its step 1 (the last reader of R1).  Likewise
// R2.  Each mbarrier is re-armed right after its wait, before this CTA
// sends anything that could let a sender run ahead.  (A two-buffer variant
// with register-staged pushes measured 7% slower at the same occupancy.)
template <typename T, int S, int C>
__global__ void __launch_bounds__(ClusterGeo<T, S, C>::NT, ClusterGeo<T, S, C>::MINB)
k_hidft_cluster(const PlanArgs args, const int32_t* __restrict__ inv1) {
  using CG = ClusterGeo<T, S, C>;
  constexpr int LC = CG::LC, SL = CG::SL, AL = CG::AL, PER = CG::PER, NT = CG::NT, EPU = CG::EPU;
  using G = typename CG::G;
  constexpr int LNT = ilog2c(NT);
  constexpr uint32_t BYTES = AL * sizeof(Cx<T>);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* W = reinterpret_cast<Cx<T>*>(smem_raw);
  Cx<T>* R1 = W + AL;
  Cx<T>* R2 = R1 + AL;
  __shared__ __align__(8) unsigned long long s_mbar[2];
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  const int t = threadIdx.x;
  const Cx<T>* tw = reinterpret_cast<const Cx<T>*>(args.tw);
  // pre-gathered rows: slot order (identity 1) or sorted order (identity 2,
  // coalesced: sorted position u reads row[u])
  const uint32_t nmask = args.identity ? (uint32_t)((1u << S) - 1u)
                                       : ((args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u));
  const uint32_t mb0 = smem_addr(&s_mbar[0]), mb1 = smem_addr(&s_mbar[1]);
  const uint32_t r1_addr = smem_addr(R1), r2_addr = smem_addr(R2);
  if (t == 0) {
    mbar_init(mb0, 1);
    mbar_init(mb1, 1);
    mbar_expect_tx(mb0, BYTES);
    mbar_expect_tx(mb1, BYTES);
  }
  cluster.sync();  // barrier inits visible cluster-wide
#define SFFT_D(i)                                                 \
  (args.identity == 1   ? (1u << (i))                             \
   : args.identity == 2 ? (1u << (S - 1 - (i)))                   \
                        : (1u << (args.M - 1 - args.used[(i)])))
  uint32_t offt = args.negshift;
#pragma unroll
  for (int j = 0; j < LNT; ++j)
    if ((t >> j) & 1) offt += SFFT_D(S - 1 - j);
#pragma unroll
  for (int j = 0; j < LC; ++j)
    if ((q >> j) & 1) offt += SFFT_D(S - 1 - (SL + j));
  uint32_t dx[G::LE > 0 ? G::LE : 1];
#pragma unroll
  for (int j = 0; j < G::LE; ++j) dx[j] = SFFT_D(S - 1 - (LNT + j));
#undef SFFT_D
  const T scale = (T)args.scale1;
  const int64_t ncl = gridDim.x / C;
  const int64_t nrows = args.B * args.nshift;
  // gather sorted positions u = x*NT + t of output row bb (signal bb / nshift,
  // shift shift0 + bb % nshift) into v
  auto gather_sorted = [&](Cx<T>(&v)[G::E], int64_t bb) {
    const int64_t bs = bb / args.nshift;
    const uint32_t sh = (uint32_t)(bb % args.nshift);
#pragma unroll
    for (int x = 0; x < G::E; ++x) {
      uint32_t off = offt - sh;
#pragma unroll
      for (int j = 0; j < G::LE; ++j)
        if ((x >> j) & 1) off += dx[j];
      if (sizeof(T) == 8 && args.in_c64) {
        const Cx<float> s = load_sample(reinterpret_cast<const Cx<float>*>(args.sig) + bs * args.ld + (off & nmask));
        v[x] = Cx<T>{(T)s.x, (T)s.y};
      } else {
        v[x] = load_sample(reinterpret_cast<const Cx<T>*>(args.sig) + bs * args.ld + (off & nmask));
      }
    }
  };
  Cx<T> v[G::E];
  if (blockIdx.x / C < nrows) gather_sorted(v, blockIdx.x / C);
  uint32_t par = 0;
  for (int64_t b = blockIdx.x / C; b < nrows; b += ncl, par ^= 1u) {
    SFFT_STAMP(0);
    // ---- 0. stage by owner (XOR by owner: conflict-free), push to R1s
#pragma unroll
    for (int x = 0; x < G::E; ++x) {
      const uint32_t u = (uint32_t)(x * NT + t);
      const uint32_t r = brev_s<LC>(u & (C - 1));
      const uint32_t i = brev_s<SL>(u) & (PER - 1);
      W[r * PER + (i ^ r)] = v[x];
    }
    __syncthreads();
    for (int w = t; w < AL / EPU; w += NT) {
      const int j0 = w * EPU;
      const int r = j0 / PER, jj = j0 % PER;
      const int i0 = jj ^ r;  // staged element i0 (and its pair partner i0^1)
      Cx<T> e0 = W[j0], e1 = W[j0 + EPU - 1];
      if (EPU == 2 && (i0 & 1)) { const Cx<T> tmp = e0; e0 = e1; e1 = tmp; }
      const uint32_t dst = r1_addr + (uint32_t)((q * PER + (i0 & ~(EPU - 1))) * sizeof(Cx<T>));
      st_async16(cluster_addr(dst, r), e0, e1, cluster_addr(mb0, r));
    }
    __syncthreads();  // W free for the local stages
    SFFT_STAMP(1);
    mbar_wait(mb0, par);
    SFFT_STAMP(2);
    if (t == 0) mbar_expect_tx(mb0, BYTES);  // arm for the next signal
    // ---- 1. local stages; pass 0 reads R1[src][i] for local slot (i << LC) | brev(src)
#pragma unroll
    for (int x = 0; x < G::E; ++x) {
      const int al = x + t * G::E;
      v[x] = R1[brev_s<LC>((uint32_t)(al & (C - 1))) * PER + (al >> LC)];
    }
    butterfly<T, SL, false, CG::EC>(v, t, W, tw);
    SFFT_STAMP(3);
    // ---- 2. push local range [q'*PER, (q'+1)*PER) to CTA q'
    for (int w = t; w < AL / EPU; w += NT) {
      const int j0 = w * EPU;
      const int qd = j0 / PER, ii = j0 % PER;
      const int p0 = swz<T, SL>(j0);
      const Cx<T> e0 = W[p0], e1 = W[p0 ^ (EPU - 1)];
      const uint32_t dst = r2_addr + (uint32_t)((q * PER + ii) * sizeof(Cx<T>));
      st_async16(cluster_addr(dst, qd), e0, e1, cluster_addr(mb1, qd));
    }
    // prefetch the next signal's samples: their latency hides behind steps 2-3
    if (b + ncl < nrows) gather_sorted(v, b + ncl);
    mbar_wait(mb1, par);
    SFFT_STAMP(4);
    if (t == 0) mbar_expect_tx(mb1, BYTES);
    // ---- 3. stages SL+1..S for local indices al = q*PER + i
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + b * args.ld1;
    Cx<T>* o2 = args.out2 ? reinterpret_cast<Cx<T>*>(args.out2) + b * args.ld2 : nullptr;
    for (int i = t; i < PER; i += NT) {
      const int al = q * PER + i;
      Cx<T> w[C];
#pragma unroll
      for (int x = 0; x < C; ++x) w[x] = R2[x * PER + i];
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        Cx<T> twj[C / 2];
#pragma unroll
        for (int x = 0; x < C / 2; ++x)
          if (x < (1 << j)) twj[x] = tw[(1 << (SL + j)) - 1 + al + (x << SL)];
#pragma unroll
        for (int x = 0; x < C; ++x) {
          if (x & (1 << j)) continue;
          bfly(w[x], w[x | (1 << j)], twj[x & ((1 << j) - 1)]);
        }
      }
#pragma unroll
      for (int x = 0; x < C; ++x) {
        const int a = al + x * AL;
        const int pos = inv1 ? __ldg(inv1 + a) : a;
        if (pos >= 0) o1[pos] = cscale(w[x], scale);
        if (o2) o2[a] = w[x];
      }
    }
    __syncthreads();  // W staging of the next signal after every push read W
    SFFT_STAMP(5);
  }
  cluster.sync();  // no CTA leaves while peers may still push into it
}

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

template <typename T, int S, bool PS> constexpr size_t fused_smem() {
  using G = Geo<T, S>;
  constexpr size_t NP = PS ? G::SPC : 1;
  return (size_t)G::SPC * G::A * sizeof(Cx<T>) + NP * (G::A > 1 ? G::A - 1 : 1) * sizeof(Cx<T>) +
         NP * G::A * sizeof(int);
}

// PER_SIGNAL: one CTA per SPC signals, each group derives its own support's
// plan on chip, then gathers, transforms and stores.  Shared support: CTAs
// are persistent, build the one plan once and loop over signal groups.
template <typename T, int S, bool PER_SIGNAL>
__global__ void __launch_bounds__(Geo<T, S>::NT, Geo<T, S>::MINB)
k_fused_to_dft(const FusedArgs args) {
  using G = Geo<T, S>;
  constexpr int A = G::A;
  constexpr int NP = PER_SIGNAL ? G::SPC : 1;  // plans held per CTA
  constexpr int TWN = A > 1 ? A - 1 : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sdata = reinterpret_cast<Cx<T>*>(smem_raw);            // SPC * A
  Cx<T>* stw_all = sdata + G::SPC * A;                          // NP * TWN
  int* spats_all = reinterpret_cast<int*>(stw_all + NP * TWN);  // NP * A
  __shared__ int sctl[NP][2 + (S > 0 ? S : 1)];

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
      if (live && t == 0 && args.status) args.status[b] = st;
    }
    const bool ok = live && st == 0;
    Cx<T> v[G::E];
    if (ok) {
      uint32_t d[S > 0 ? S : 1];
#pragma unroll
      for (int i = 0; i < S; ++i) d[i] = args.identity ? (1u << i) : (1u << (args.M - 1 - spiv[i]));
      const Cx<T>* row = reinterpret_cast<const Cx<T>*>(args.sig) + b * args.ld;
      gather<T, S>(v, t, row, d, 0u, args.identity ? (uint32_t)(A - 1) : nmask);
    } else {
#pragma unroll
      for (int x = 0; x < G::E; ++x) v[x] = Cx<T>{T(0), T(0)};
    }
    butterfly<T, S>(v, t, sd, tw);
    if (ok) {
      Cx<T>* o = reinterpret_cast<Cx<T>*>(args.out) + b * args.ld_out;
      for (int i = t; i < A; i += G::TPS) o[i] = cscale(sd[swz<T, S>(pats[i])], scale);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ launchers ---

// Per (kernel, device): opt in to the full dynamic shared memory and cache
// the occupancy (resident CTAs per SM).
static std::mutex g_kmu;
static std::map<std::pair<const void*, int>, int> g_occ;

template <typename K>
static int kernel_occupancy(K kernel, int nt, size_t smem, int* occ) {
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  {
    std::lock_guard<std::mutex> lk(g_kmu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) {
      *occ = it->second;
      return SFFT_OK;
    }
  }
  SFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int o = 0;
  SFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, nt, smem));
  if (o < 1) return fail(SFFT_ERR_UNSUPPORTED, "kernel does not fit on an SM");
  std::lock_guard<std::mutex> lk(g_kmu);
  g_occ[key] = o;
  *occ = o;
  return SFFT_OK;
}

template <typename T, int S>
static int run_plan_kernel(const PlanArgs& a, cudaStream_t st) {
  using G = Geo<T, S>;
  constexpr size_t smem = plan_smem<T, S>();
  static_assert(smem <= 227 * 1024, "plan kernel smem");
  auto kern = k_hidft_plan<T, S>;
  int occ = 0;
  int rc = kernel_occupancy(kern, G::NT, smem, &occ);
  if (rc) return rc;
  const int64_t ngroups = (a.B * a.nshift + G::SPC - 1) / G::SPC;
  if (ngroups > 0x7fffffff) return fail(SFFT_ERR_UNSUPPORTED, "batch too large for one launch");
  kern<<<(unsigned)ngroups, G::NT, smem, st>>>(a);
  SFFT_CUDA(cudaGetLastError());
  return SFFT_OK;
}

template <typename T, int S, bool PS>
static int run_fused_kernel(const FusedArgs& a, cudaStream_t st) {
  using G = Geo<T, S>;
  constexpr size_t smem = fused_smem<T, S, PS>();
  static_assert(smem <= 227 * 1024, "fused kernel smem");
  auto kern = k_fused_to_dft<T, S, PS>;
  int occ = 0;
  int rc = kernel_occupancy(kern, G::NT, smem, &occ);
  if (rc) return rc;
  const int64_t ngroups = (a.B + G::SPC - 1) / G::SPC;
  int64_t grid = PS ? ngroups : std::min<int64_t>(ngroups, (int64_t)num_sms() * occ);
  if (grid > 0x7fffffff) return fail(SFFT_ERR_UNSUPPORTED, "batch too large for one launch");
  kern<<<(unsigned)std::max<int64_t>(grid, 1), G::NT, smem, st>>>(a);
  SFFT_CUDA(cudaGetLastError());
  return SFFT_OK;
}

template <typename T, int S, int C>
static int run_cluster_kernel(const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  using CG = ClusterGeo<T, S, C>;
  constexpr size_t smem = CG::SMEM;
  static_assert(smem <= 227 * 1024, "cluster kernel smem");
  auto kern = k_hidft_cluster<T, S, C>;
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(CG::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = 0;
  {
    std::lock_guard<std::mutex> lk(g_kmu);
    const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
    auto it = g_occ.find(key);
    if (it == g_occ.end()) {
      SFFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      if (C > 8) SFFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cfg.gridDim = dim3(C);
      SFFT_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
      if (max_clusters < 1) return fail(SFFT_ERR_UNSUPPORTED, "cluster does not fit on the device");
      g_occ[key] = max_clusters;
    } else {
      max_clusters = it->second;
    }
  }
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(a.B * a.nshift, max_clusters));
  cfg.gridDim = dim3((unsigned)(ncl * C));
  SFFT_CUDA(cudaLaunchKernelEx(&cfg, kern, a, inv1));
  return SFFT_OK;
}

// ------------------------------------------ two-pass split for large A ---
//
// 2^s slots beyond one SM (configs 5/6) run as two kernels per chunk of
// rows, exchanging through an L2-resident scratch instead of DSMEM:
//
//  front (k_split_front): stage k pairs slot bit k-1, i.e. sorted-order bit
//    s-k, so the first lc stages pair samples 2^(s-lc), 2^(s-lc+1), ...
//    apart in SORTED order.  A thread owns one sorted low position p and
//    its 2^lc partners u = x*2^(s-lc) + p, loads them (warps read
//    consecutive p: contiguous runs of the pattern, full lines), runs the
//    lc stages in registers (the 2^lc - 1 twiddles depend only on x), and
//    stores value x to scratch block x at position p (coalesced).
//  back (k_split_back): block t = the sorted range [t*2^(s-lc), ...) =
//    the slots whose low lc bits are brev(t); its remaining s - lc stages
//    pair bits lc.. s-1 only, i.e. they are local.  One CTA per (row, t)
//    loads the block (coalesced) into shared memory at slot positions,
//    runs the single-CTA butterfly with the block's twiddle slice
//    (plan->d_tw_blk) and stores through the block-major inverse map.
//
// Chunks of rows keep the scratch (rows x 2^s complex) within ~32 MiB so it
// stays in L2 between the two kernels: HBM sees the samples once and the
// results once (measured L2-resident streaming: ~12 TB/s read, ~7 TB/s write,
// tools/l2_probe.cu).
template <int B>
__host__ __device__ constexpr uint32_t brev_c(uint32_t x) {
  uint32_t r = 0;
  for (int i = 0; i < B; ++i) r |= ((x >> i) & 1u) << (B - 1 - i);
  return r;
}

template <typename T, int S, int LC>
struct SplitGeo {
  static constexpr int SL = S - LC, EX = 1 << LC;
  static constexpr int NT1 = 256;                    // front: threads per CTA
  static constexpr int NSEG = (1 << SL) / NT1;       // front CTAs per row
  using G = Geo<T, SL>;                              // back: single-CTA geometry
  static_assert(G::SPC == 1, "back pass: one block per CTA");
#ifndef SFFT_BACK_BMIN
#define SFFT_BACK_BMIN 2
#endif
  static constexpr int BMIN = G::NT <= 256 ? SFFT_BACK_BMIN : 1;  // back: CTAs per SM
  // back: double-buffered rows + inverse map in shared memory when 1-2 CTAs
  // fit per SM; one row buffer (more CTAs hide each other's loads) otherwise
  static constexpr bool DB = BMIN < 3;
  static constexpr size_t SMEM = (size_t)(1 << SL) * ((DB ? 3 : 2) * sizeof(Cx<T>) + (DB ? sizeof(int32_t) : 0));
};

template <typename T, int S, int LC>
__global__ void __launch_bounds__(256) k_split_front(const PlanArgs args, Cx<T>* __restrict__ scratch,
                                                     int64_t row0) {
  using SG = SplitGeo<T, S, LC>;
  constexpr int SL = SG::SL, EX = SG::EX;
  const int64_t rr = blockIdx.x / SG::NSEG;  // row within the chunk
  const uint32_t p = (blockIdx.x % SG::NSEG) * SG::NT1 + threadIdx.x;
  const int64_t r = row0 + rr;               // output row
  const int64_t bs = (args.debug_skip & 16) ? (r & 1) : r / args.nshift;  // bit 4: footprint probe
  // slot bit i -> sample stride d_i (hidft.py:155-158), or the pre-gathered layouts
  uint32_t d[S];
#pragma unroll
  for (int i = 0; i < S; ++i)
    d[i] = args.identity == 1   ? (1u << i)
           : args.identity == 2 ? (1u << (S - 1 - i))
                                : (1u << (args.M - 1 - args.used[i]));
  const uint32_t nmask = args.identity ? (uint32_t)((1u << S) - 1u)
                                       : ((args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u));
  // sorted bit j <-> slot bit S-1-j
  uint32_t off = args.identity ? 0u : ((args.negshift - (uint32_t)(r % args.nshift)) & nmask);
#pragma unroll
  for (int j = 0; j < SL; ++j)
    if ((p >> j) & 1u) off += d[S - 1 - j];
  Cx<T> v[EX];
#pragma unroll
  for (int x = 0; x < EX; ++x) {
    uint32_t o = off;
#pragma unroll
    for (int j = 0; j < LC; ++j)
      if ((x >> j) & 1) o += d[LC - 1 - j];
    if (sizeof(T) == 8 && args.in_c64) {
      const Cx<float> sv = load_sample(reinterpret_cast<const Cx<float>*>(args.sig) + bs * args.ld + (o & nmask));
      v[x] = Cx<T>{(T)sv.x, (T)sv.y};
    } else {
      v[x] = load_sample(reinterpret_cast<const Cx<T>*>(args.sig) + bs * args.ld + (o & nmask));
    }
  }
  // stages 1..LC: stage k pairs slot bit k-1 = x bit LC-k; twiddle index
  // a mod 2^(k-1) = brev_LC(x) mod 2^(k-1) (hidft.py:160-167)
  const Cx<T>* tw = reinterpret_cast<const Cx<T>*>(args.tw);
#pragma unroll
  for (int k = 1; k <= LC; ++k) {
    const int lb = LC - k;
#pragma unroll
    for (int x = 0; x < EX; ++x) {
      if (x & (1 << lb)) continue;
      const uint32_t h = brev_c<LC>((uint32_t)x) & ((1u << (k - 1)) - 1u);
      bfly(v[x], v[x | (1 << lb)], tw[(1 << (k - 1)) - 1 + h]);
    }
  }
  Cx<T>* dst = scratch + ((rr * EX) << SL) + p;
#pragma unroll
  for (int x = 0; x < EX; ++x) dst[(int64_t)x << SL] = v[x];
}

// cp.async of one element (8 B c64 / 16 B c128) global -> shared, L2 only
__device__ __forceinline__ void cp_async_elem(void* sdst, const Cx<float>* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(smem_addr(sdst)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_elem(void* sdst, const Cx<double>* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr(sdst)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// Persistent: CTA i serves block tb = i mod 2^lc for rows i / 2^lc, + nper, ...
// of the chunk.  The block's twiddle slice and inverse map are staged in
// shared memory once (the same for every row); rows are double-buffered:
// the next row's block is copied (cp.async, straight into its bit-reversed
// slot positions) while this row's butterfly and stores run.
template <typename T, int S, int LC>
__global__ void __launch_bounds__(SplitGeo<T, S, LC>::G::NT, SplitGeo<T, S, LC>::BMIN)
k_split_back(const PlanArgs args, const Cx<T>* __restrict__ scratch, int64_t row0, int64_t nrows, int nper,
             const Cx<T>* __restrict__ tw_blk, const int32_t* __restrict__ inv_blk) {
  using SG = SplitGeo<T, S, LC>;
  using G = typename SG::G;
  constexpr int SL = SG::SL, EX = SG::EX, AL = 1 << SL, NT = G::NT, PT = AL / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr bool DB = SG::DB;
  Cx<T>* sbuf = reinterpret_cast<Cx<T>*>(smem_raw);  // (DB ? 2 : 1) x AL
  Cx<T>* stw = sbuf + (DB ? 2 : 1) * AL;
  int32_t* sinv = reinterpret_cast<int32_t*>(stw + AL);  // DB only
  const int tid = threadIdx.x;
  const int tb = blockIdx.x % EX;
  const int64_t first = blockIdx.x / EX;
  if (first >= nrows) return;
  // block tb in sorted order: position j holds local slot brev_SL(j)
  auto issue = [&](int64_t rr, Cx<T>* dst) {
    const Cx<T>* src = scratch + ((rr * EX + tb) << SL);
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int j = tid + n * NT;
      cp_async_elem(dst + swz<T, SL>((int)(__brev((uint32_t)j) >> (32 - SL))), src + j);
    }
    cp_async_commit();
  };
  issue(first, sbuf);
  {
    const Cx<T>* twg = tw_blk + (int64_t)tb * (AL - 1);
    Cx<T> t[PT];
    int32_t e[PT];
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int i = tid + n * NT;
      t[n] = i < AL - 1 ? twg[i] : Cx<T>{T(0), T(0)};
      e[n] = (DB && inv_blk) ? __ldg(inv_blk + ((int64_t)tb << SL) + i) : 0;
    }
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int i = tid + n * NT;
      if (i < AL - 1) stw[i] = t[n];
      if (DB) sinv[i] = e[n];
    }
  }
  const T scale = (T)args.scale1;
  const uint32_t lowbits = brev_c<LC>((uint32_t)tb);  // fixed low slot bits of this block
  int cur = 0;
  for (int64_t rr = first; rr < nrows; rr += nper, cur ^= 1) {
    const int64_t r = row0 + rr;
    Cx<T>* sd = sbuf + (DB ? cur * AL : 0);
    if (!DB) {
      if (rr != first) issue(rr, sbuf);
      cp_async_wait<0>();
    } else if (rr + nper < nrows) {
      issue(rr + nper, sbuf + (cur ^ 1) * AL);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // this row's block (and the tables) visible to all threads
    Cx<T> v[G::E];
    if (!(args.debug_skip & 4)) butterfly<T, SL, true>(v, tid, sd, stw);
    Cx<T> val[PT];
    int32_t e[PT];
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int l = tid + n * NT;
      val[n] = sd[swz<T, SL>(l)];
      e[n] = DB ? sinv[l] : (inv_blk ? __ldg(inv_blk + ((int64_t)tb << SL) + l) : 0);
    }
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + r * args.ld1;
    if (args.debug_skip & 2) {
#pragma unroll
      for (int n = 0; n < PT; ++n)
        if (e[n] == -7) o1[n] = val[n];
    } else if (args.debug_skip & 8) {  // coalesced stores (timing probe only)
#pragma unroll
      for (int n = 0; n < PT; ++n) o1[(tb << SL) + tid + n * NT] = val[n];
    } else if (inv_blk) {
#pragma unroll
      for (int n = 0; n < PT; ++n)
        if (e[n] >= 0) o1[e[n]] = cscale(val[n], scale);
    } else {  // slot order output
#pragma unroll
      for (int n = 0; n < PT; ++n) o1[((uint32_t)(tid + n * NT) << LC) | lowbits] = cscale(val[n], scale);
    }
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + r * args.ld2;
#pragma unroll
      for (int n = 0; n < PT; ++n) o2[((uint32_t)(tid + n * NT) << LC) | lowbits] = val[n];
    }
    __syncthreads();  // sd is refilled (two rows on when double-buffered)
  }
}

// ------------------------------------------------ fused persistent split ---
//
// One cooperative (all CTAs co-resident) launch runs both passes as a
// software pipeline.  CTAs form groups of 2^lc; group g owns rows g, g + G,
// ...; CTA q of a group does front segment q and back block q of each of
// the group's rows.  Per row i a CTA: issues the cp.async gather of row
// i+1's front segment into shared memory; waits (global counter, acquire)
// until the group's 2^lc front segments of row i are in the scratch ring;
// stages its back block; runs the butterfly and the scattered stores
// (row i+1's samples arrive meanwhile); then finishes row i+1's front
// stages and publishes them (release).  The ring (2 rows per group) stays
// in L2, so HBM sees the samples once and the results once, and the HBM
// gather overlaps the shared-memory butterfly of the previous row.
static int scratch_pool(int dev, cudaMemPool_t* pool);

struct SplitSync {
  unsigned int* front;  // [G][2]: front segments stored, cumulative per slot
  unsigned int* back;   // [G][2]: back blocks staged (slot consumed), cumulative
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// thread 0 waits for *p >= target; co-residency (cooperative launch) makes
// this deadlock-free; the bound only turns a logic error into a fault
__device__ __forceinline__ void wait_count(const unsigned int* p, unsigned int target) {
  if (threadIdx.x == 0) {
    unsigned int spins = 0;
    while (ld_acquire_gpu(p) < target) {
      __nanosleep(40);
      if (++spins > (1u << 28)) __trap();
    }
  }
  __syncthreads();
}
__device__ __forceinline__ Cx<float> ld_cg(const Cx<float>* p) {
  Cx<float> r;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ Cx<double> ld_cg(const Cx<double>* p) {
  Cx<double> r;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

template <typename T, int S, int LC, typename In>
struct FusedSplitGeo {
  using SG = SplitGeo<T, S, LC>;
  using G = typename SG::G;
  static constexpr int SL = SG::SL, EX = SG::EX, AL = 1 << SL, NT = G::NT;
  static constexpr int PQ = AL / EX;  // front positions per CTA
  static constexpr size_t SMEM = (size_t)AL * (2 * sizeof(Cx<T>) + sizeof(int32_t) + sizeof(Cx<In>));
  static constexpr int BMIN = SMEM * 2 <= 227 * 1024 && NT <= 256 ? 2 : 1;
};

template <typename T, int S, int LC, typename In>
__global__ void __launch_bounds__(FusedSplitGeo<T, S, LC, In>::NT, FusedSplitGeo<T, S, LC, In>::BMIN)
k_split_fused(const PlanArgs args, Cx<T>* __restrict__ ring, SplitSync sync, const Cx<T>* __restrict__ tw_blk,
              const int32_t* __restrict__ inv_blk) {
  using FG = FusedSplitGeo<T, S, LC, In>;
  using G = typename FG::G;
  constexpr int SL = FG::SL, EX = FG::EX, AL = FG::AL, NT = FG::NT, PQ = FG::PQ, PT = AL / NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sd = reinterpret_cast<Cx<T>*>(smem_raw);
  Cx<T>* stw = sd + AL;
  int32_t* sinv = reinterpret_cast<int32_t*>(stw + AL);
  Cx<In>* sf = reinterpret_cast<Cx<In>*>(sinv + AL);  // front samples [x][p - q*PQ]
  const int tid = threadIdx.x;
  const int q = blockIdx.x % EX;
  const int64_t g = blockIdx.x / EX, ngroups = gridDim.x / EX;
  const int64_t rows = args.B * args.nshift;
  if (g >= rows) return;
  const int64_t nmine = (rows - g + ngroups - 1) / ngroups;
  Cx<T>* myring = ring + (g * 2) * ((int64_t)EX << SL);
  unsigned int* fcnt = sync.front + g * 2;
  unsigned int* bcnt = sync.back + g * 2;

  // sample strides: slot bit i -> d_i (hidft.py:155-158) or pre-gathered layouts
  uint32_t d[S];
#pragma unroll
  for (int i = 0; i < S; ++i)
    d[i] = args.identity == 1   ? (1u << i)
           : args.identity == 2 ? (1u << (S - 1 - i))
                                : (1u << (args.M - 1 - args.used[i]));
  const uint32_t nmask = args.identity ? (uint32_t)((1u << S) - 1u)
                                       : ((args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u));
  // front gather of row i: cp.async of this CTA's PQ positions x 2^lc
  // partners; the offsets (without the row's shift) are fixed per thread
  constexpr int FPT = EX * PQ / NT;  // front samples per thread
  static_assert(EX * PQ % NT == 0, "front split");
  uint32_t foff[FPT];
#pragma unroll
  for (int n = 0; n < FPT; ++n) {
    const int idx = tid + n * NT;
    const int x = idx / PQ;
    const uint32_t p = (uint32_t)(q * PQ + idx % PQ);
    uint32_t o = 0;
    for (int j = 0; j < SL; ++j)
      if ((p >> j) & 1u) o += d[S - 1 - j];
    for (int j = 0; j < LC; ++j)
      if ((x >> j) & 1) o += d[LC - 1 - j];
    foff[n] = o;
  }
  auto front_issue = [&](int64_t i) {
    const int64_t r = g + i * ngroups;
    const int64_t bs = r / args.nshift;
    const uint32_t base = args.identity ? 0u : ((args.negshift - (uint32_t)(r % args.nshift)) & nmask);
    const Cx<In>* row = reinterpret_cast<const Cx<In>*>(args.sig) + bs * args.ld;
#pragma unroll
    for (int n = 0; n < FPT; ++n) cp_async_elem(sf + tid + n * NT, row + ((base + foff[n]) & nmask));
    cp_async_commit();
  };
  // front stages of row i (samples in sf), stored to the ring and published
  auto front_finish = [&](int64_t i) {
    const int slot = (int)(i & 1);
    Cx<T>* dst = myring + (int64_t)slot * ((int64_t)EX << SL);
    // slot reuse: row i-2's blocks must have been staged by the whole group
    if (i >= 2) wait_count(bcnt + slot, (unsigned)(EX * (i / 2)));
    const Cx<T>* tw = reinterpret_cast<const Cx<T>*>(args.tw);
    for (int pl = tid; pl < PQ; pl += NT) {
      Cx<T> v[EX];
#pragma unroll
      for (int x = 0; x < EX; ++x) {
        const Cx<In> sv = sf[x * PQ + pl];
        v[x] = Cx<T>{(T)sv.x, (T)sv.y};
      }
#pragma unroll
      for (int k = 1; k <= LC; ++k) {
        const int lb = LC - k;
#pragma unroll
        for (int x = 0; x < EX; ++x) {
          if (x & (1 << lb)) continue;
          const uint32_t h = brev_c<LC>((uint32_t)x) & ((1u << (k - 1)) - 1u);
          bfly(v[x], v[x | (1 << lb)], tw[(1 << (k - 1)) - 1 + h]);
        }
      }
      const int p = q * PQ + pl;
#pragma unroll
      for (int x = 0; x < EX; ++x) dst[((int64_t)x << SL) + p] = v[x];
    }
    __syncthreads();  // every thread's stores precede thread 0's (cumulative) release
  };
  // publish row i's front segment: released late so the ring stores have
  // drained by then (the release waits for them)
  auto front_publish = [&](int64_t i) {
    if (tid == 0) red_release_gpu(fcnt + (int)(i & 1), 1u);
  };

  // tables of back block q, staged once
  {
    const Cx<T>* twg = tw_blk + (int64_t)q * (AL - 1);
    for (int i = tid; i < AL - 1; i += NT) stw[i] = twg[i];
    for (int i = tid; i < AL; i += NT) sinv[i] = inv_blk ? __ldg(inv_blk + ((int64_t)q << SL) + i) : 0;
  }
  front_issue(0);
  cp_async_wait<0>();
  __syncthreads();
  front_finish(0);
  front_publish(0);
  const T scale = (T)args.scale1;
  const uint32_t lowbits = brev_c<LC>((uint32_t)q);
  SFFT_ACC_INIT();
  for (int64_t i = 0; i < nmine; ++i) {
    const int64_t r = g + i * ngroups;
    const int slot = (int)(i & 1);
    const bool more = i + 1 < nmine;
    if (more) front_issue(i + 1);  // samples of the next row fly during this row's back pass
    if (i > 0) front_publish(i);   // row i's front segment, finished last iteration
    SFFT_ACC(0);
    wait_count(fcnt + slot, (unsigned)(EX * (i / 2 + 1)));
    SFFT_ACC(1);
    {  // stage back block q of row i (sorted order -> slot positions), L2 loads
      const Cx<T>* src = myring + (int64_t)slot * ((int64_t)EX << SL) + ((int64_t)q << SL);
      Cx<T> t[PT];
#pragma unroll
      for (int n = 0; n < PT; ++n) t[n] = ld_cg(src + tid + n * NT);
#pragma unroll
      for (int n = 0; n < PT; ++n) {
        const int j = tid + n * NT;
        sd[swz<T, SL>((int)(__brev((uint32_t)j) >> (32 - SL)))] = t[n];
      }
    }
    __syncthreads();
    if (tid == 0) red_release_gpu(bcnt + slot, 1u);  // slot may be refilled once all 2^lc staged
    SFFT_ACC(2);
    Cx<T> v[G::E];
    butterfly<T, SL, true>(v, tid, sd, stw);
    SFFT_ACC(3);
    Cx<T> val[PT];
    int32_t e[PT];
#pragma unroll
    for (int n = 0; n < PT; ++n) {
      const int l = tid + n * NT;
      val[n] = sd[swz<T, SL>(l)];
      e[n] = sinv[l];
    }
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + r * args.ld1;
    if (inv_blk) {
#pragma unroll
      for (int n = 0; n < PT; ++n)
        if (e[n] >= 0) o1[e[n]] = cscale(val[n], scale);
    } else {
#pragma unroll
      for (int n = 0; n < PT; ++n) o1[((uint32_t)(tid + n * NT) << LC) | lowbits] = cscale(val[n], scale);
    }
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + r * args.ld2;
#pragma unroll
      for (int n = 0; n < PT; ++n) o2[((uint32_t)(tid + n * NT) << LC) | lowbits] = val[n];
    }
    SFFT_ACC(4);
    if (more) {
      cp_async_wait<0>();
      __syncthreads();  // next row's samples landed; sd reads of this row done
      SFFT_ACC(5);
      front_finish(i + 1);
      SFFT_ACC(6);
    } else {
      __syncthreads();
    }
  }
}

template <typename T, int S, int LC, typename In>
static int run_split_fused(const sfft_plan* p, const PlanArgs& a, const int32_t* inv_blk, cudaStream_t st) {
  using FG = FusedSplitGeo<T, S, LC, In>;
  auto kern = k_split_fused<T, S, LC, In>;
  static_assert(FG::SMEM <= 227 * 1024, "fused split smem");
  int occ = 0, rc;
  if ((rc = kernel_occupancy(kern, FG::NT, FG::SMEM, &occ))) return rc;
  const int64_t rows = a.B * a.nshift;
  if (rows == 0) return SFFT_OK;
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>(rows, (int64_t)num_sms() * occ / FG::EX));
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  if ((rc = scratch_pool(dev, &pool))) return rc;
  const size_t ring_bytes = (size_t)G * 2 * (sizeof(Cx<T>) << S);
  const size_t sync_bytes = (size_t)G * 4 * sizeof(unsigned int);
  void* buf = nullptr;
  SFFT_CUDA(cudaMallocFromPoolAsync(&buf, ring_bytes + sync_bytes, pool, st));
  unsigned int* cnt = reinterpret_cast<unsigned int*>((char*)buf + ring_bytes);
  cudaError_t e = cudaMemsetAsync(cnt, 0, sync_bytes, st);
  if (e == cudaSuccess) {
    PlanArgs aa = a;
    Cx<T>* ring = reinterpret_cast<Cx<T>*>(buf);
    SplitSync sy{cnt, cnt + 2 * G};
    const Cx<T>* twb = reinterpret_cast<const Cx<T>*>(p->d_tw_blk);
    void* params[] = {(void*)&aa, (void*)&ring, (void*)&sy, (void*)&twb, (void*)&inv_blk};
    e = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)(G * FG::EX)), dim3(FG::NT), params, FG::SMEM,
                                    st);
  }
  cudaFreeAsync(buf, st);
  if (e != cudaSuccess) return cuda_fail(e, "fused split launch");
  return SFFT_OK;
}

// stream-ordered scratch from a library-owned pool that keeps its memory
static int scratch_pool(int dev, cudaMemPool_t* pool) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) {
    *pool = it->second;
    return SFFT_OK;
  }
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t p;
  SFFT_CUDA(cudaMemPoolCreate(&p, &props));
  uint64_t keep = ~0ull;
  SFFT_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
  pools[dev] = p;
  *pool = p;
  return SFFT_OK;
}

// rows per chunk of the two-kernel split: scratch up to SFFT_SPLIT_SCRATCH_MB
// (default 128 MiB, measured best for config 5, tools/cfg5_sweep.sh), rounded
// to a multiple of the back pass's rows per wave so its persistent CTAs all
// get the same number of rows
static int64_t split_chunk_rows(int64_t rows, size_t row_bytes, int occ, int ex) {
  static const int64_t scr_mb = [] {
    const char* e = getenv("SFFT_SPLIT_SCRATCH_MB");
    return (int64_t)(e ? std::max(1, atoi(e)) : 128);
  }();
  const int64_t per_wave = std::max<int64_t>(1, (int64_t)num_sms() * occ / ex);
  int64_t chunk = std::max<int64_t>(1, (scr_mb << 20) / (int64_t)row_bytes);
  return std::max<int64_t>(1, std::min<int64_t>(rows, (chunk + per_wave - 1) / per_wave * per_wave));
}

static bool split_fused_selected() {
  static const bool fused = [] { const char* e = getenv("SFFT_SPLIT"); return e && std::string(e) == "fused"; }();
  return fused;
}

// kernel launches run_split issues for `rows` rows (sfft_launch_count)
template <typename T, int S, int LC>
static int split_launches(int64_t rows, int64_t* n) {
  using SG = SplitGeo<T, S, LC>;
  if (split_fused_selected()) {
    *n = rows > 0 ? 1 : 0;
    return SFFT_OK;
  }
  int occ = 0;
  int rc = kernel_occupancy(k_split_back<T, S, LC>, SG::G::NT, SG::SMEM, &occ);
  if (rc) return rc;
  const int64_t chunk = split_chunk_rows(rows, sizeof(Cx<T>) << S, occ, SG::EX);
  *n = rows > 0 ? 2 * ((rows + chunk - 1) / chunk) : 0;
  return SFFT_OK;
}

template <typename T, int S, int LC>
static int run_split(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  using SG = SplitGeo<T, S, LC>;
  using G = typename SG::G;
  if (p->split_lc != LC || !p->d_tw_blk) return fail(SFFT_ERR_INVALID, "plan has no split tables");
  const int32_t* inv_blk = inv1 == p->d_inv_elem ? p->d_inv_elem_blk
                           : inv1 == p->d_inv_node ? p->d_inv_node_blk
                                                   : nullptr;
  if (inv1 && !inv_blk) return fail(SFFT_ERR_INVALID, "no block-major map for this output");
  // the fused persistent pipeline measured slower than two launches on config 5
  // (200 vs 185 us, tools/split_time.py); kept selectable for study
  if (split_fused_selected()) {
    if (sizeof(T) == 8 && a.in_c64) return run_split_fused<T, S, LC, float>(p, a, inv_blk, st);
    return run_split_fused<T, S, LC, T>(p, a, inv_blk, st);
  }
  auto front = k_split_front<T, S, LC>;
  auto back = k_split_back<T, S, LC>;
  PlanArgs ab = a;
  static const int dbg = [] { const char* e = getenv("SFFT_SPLIT_DEBUG"); return e ? atoi(e) : 0; }();
  ab.debug_skip = dbg;
  int occ = 0, rc;
  if ((rc = kernel_occupancy(back, G::NT, SG::SMEM, &occ))) return rc;
  const int64_t rows = a.B * a.nshift;
  if (rows == 0) return SFFT_OK;
  const size_t row_bytes = sizeof(Cx<T>) << S;
  const int64_t chunk = split_chunk_rows(rows, row_bytes, occ, SG::EX);
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  cudaMemPool_t pool;
  if ((rc = scratch_pool(dev, &pool))) return rc;
  void* scr = nullptr;
  SFFT_CUDA(cudaMallocFromPoolAsync(&scr, (size_t)chunk * row_bytes, pool, st));
  const Cx<T>* twb = reinterpret_cast<const Cx<T>*>(p->d_tw_blk);
  for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
    const int64_t n = std::min(chunk, rows - r0);
    front<<<(unsigned)(n * SG::NSEG), SG::NT1, 0, st>>>(ab, (Cx<T>*)scr, r0);
    const int nper = (int)std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)num_sms() * occ / SG::EX));
    back<<<(unsigned)(nper * SG::EX), G::NT, SG::SMEM, st>>>(ab, (const Cx<T>*)scr, r0, n, nper, twb, inv_blk);
  }
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scr, st);
  if (e != cudaSuccess) return cuda_fail(e, "split transform launch");
  return SFFT_OK;
}

static bool use_cluster_path() {
  static const bool v = [] {
    const char* e = getenv("SFFT_LARGE");
    return e && std::string(e) == "cluster";
  }();
  return v;
}

constexpr int kMaxFusedS_c64 = 13, kMaxFusedS_c128 = 12;

int max_supported_s(int dtype) { return dtype == SFFT_C64 ? kMaxSplitS_c64 : kMaxSplitS_c128; }

#define SFFT_CASES_12(M_, ...) \
  M_(0, __VA_ARGS__) M_(1, __VA_ARGS__) M_(2, __VA_ARGS__) M_(3, __VA_ARGS__) M_(4, __VA_ARGS__) \
  M_(5, __VA_ARGS__) M_(6, __VA_ARGS__) M_(7, __VA_ARGS__) M_(8, __VA_ARGS__) M_(9, __VA_ARGS__) \
  M_(10, __VA_ARGS__) M_(11, __VA_ARGS__) M_(12, __VA_ARGS__)

#define PLAN_CASE(S_, T_) case S_: return run_plan_kernel<T_, S_>(a, st);
#define FUSED_CASE(S_, T_, PS_) case S_: return run_fused_kernel<T_, S_, PS_>(a, st);

static int dispatch_plan(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  const int dtype = p->dtype, s = p->s;
  if (p->split_lc && !use_cluster_path()) {
    if (dtype == SFFT_C64) {
      switch (s) {
        case 15: return run_split<float, 15, 3>(p, a, inv1, st);
        case 16: return run_split<float, 16, 4>(p, a, inv1, st);
        case 17: return run_split<float, 17, 4>(p, a, inv1, st);
        default: break;
      }
    } else {
      switch (s) {
        case 14: return run_split<double, 14, 2>(p, a, inv1, st);
        case 15: return run_split<double, 15, 3>(p, a, inv1, st);
        case 16: return run_split<double, 16, 4>(p, a, inv1, st);
        default: break;
      }
    }
  }
  if (dtype == SFFT_C64) {
    switch (s) {
      SFFT_CASES_12(PLAN_CASE, float)
      PLAN_CASE(13, float)
      PLAN_CASE(14, float)
      case 15: return run_cluster_kernel<float, 15, 8>(a, inv1, st);
#ifdef SFFT_C8_FOR_S16
      case 16: return run_cluster_kernel<float, 16, 8>(a, inv1, st);
#else
      case 16: return run_cluster_kernel<float, 16, 16>(a, inv1, st);
#endif
      case 17: return run_cluster_kernel<float, 17, 16>(a, inv1, st);
      default: break;
    }
  } else {
    switch (s) {
      SFFT_CASES_12(PLAN_CASE, double)
      PLAN_CASE(13, double)
      case 14: return run_cluster_kernel<double, 14, 4>(a, inv1, st);
      case 15: return run_cluster_kernel<double, 15, 8>(a, inv1, st);
      case 16: return run_cluster_kernel<double, 16, 16>(a, inv1, st);
      default: break;
    }
  }
  return fail(SFFT_ERR_UNSUPPORTED, "2^s slots exceed the single-CTA transform (s=" +
                                        std::to_string(s) + ")");
}

template <bool PS>
static int dispatch_fused(int dtype, int s, const FusedArgs& a, cudaStream_t st) {
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
  if (plan->per_signal || !plan->split_lc || use_cluster_path() || rows == 0) return SFFT_OK;
  if (plan->dtype == SFFT_C64) {
    switch (plan->s) {
      case 15: return split_launches<float, 15, 3>(rows, launches);
      case 16: return split_launches<float, 16, 4>(rows, launches);
      case 17: return split_launches<float, 17, 4>(rows, launches);
      default: break;
    }
  } else {
    switch (plan->s) {
      case 14: return split_launches<double, 14, 2>(rows, launches);
      case 15: return split_launches<double, 15, 3>(rows, launches);
      case 16: return split_launches<double, 16, 4>(rows, launches);
      default: break;
    }
  }
  return SFFT_OK;
}

extern "C" int sfft_hidft(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
                          int64_t shift, int out_kind, void* out, int64_t ld_out, void* slot_out,
                          int64_t ld_slot, sfft_stream_t stream) {
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
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (order != SFFT_ORDER_SLOT && order != SFFT_ORDER_PATTERN) return fail(SFFT_ERR_INVALID, "unknown sample order");
  return hidft_gathered(plan, samples, B, ld, order == SFFT_ORDER_PATTERN, out_kind, out, ld_out, slot_out, ld_slot,
                        (cudaStream_t)stream);
}

extern "C" int sfft_hidft_gathered(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld,
                                   int out_kind, void* out, int64_t ld_out, void* slot_out,
                                   int64_t ld_slot, sfft_stream_t stream) {
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  return hidft_common(plan, samples, B, ld, plan->A, 0, out_kind, out, ld_out, slot_out, ld_slot, 1,
                      (cudaStream_t)stream);
}

extern "C" int sfft_plan_apply_map(const sfft_plan* plan, int out_kind, const void* slot_values,
                                   int64_t B, int64_t ld, void* out, int64_t ld_out,
                                   sfft_stream_t stream) {
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

extern "C" int sfft_hidft_to_dft_fused(const int64_t* J, int64_t k, int64_t n_supports, int M,
                                       const void* signals, int64_t B, int64_t ld, int dtype,
                                       void* out, int64_t ld_out, int32_t* status,
                                       sfft_stream_t stream) {
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
  int rc = (n_supports == 1 && B >= 1) ? dispatch_fused<false>(dtype, s, a, st)
                                       : dispatch_fused<true>(dtype, s, a, st);
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

#ifdef SFFT_PHASE_TIMING
extern "C" SFFT_API int sfft_debug_stamps(unsigned long long* out, int nblocks) {
  SFFT_CUDA(cudaDeviceSynchronize());
  SFFT_CUDA(cudaMemcpyFromSymbol(out, sfft::g_phase_stamps, sizeof(unsigned long long) * 8 * nblocks));
  return SFFT_OK;
}
extern "C" SFFT_API int sfft_debug_reset(int nblocks) {
  void* p = nullptr;
  SFFT_CUDA(cudaGetSymbolAddress(&p, sfft::g_phase_stamps));
  SFFT_CUDA(cudaMemset(p, 0, sizeof(unsigned long long) * 8 * nblocks));
  return SFFT_OK;
}
#endif
