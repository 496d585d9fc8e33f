// Two-pass split transform for 2^s beyond one CTA (configs 5/6, s = 14..17):
// a front pass runs the first lc stages across 2^lc sorted blocks in
// registers and writes an L2-resident scratch; a persistent back pass runs
// the remaining s - lc stages per block in shared memory and stores through
// the block-major inverse map.  See DESIGN.md "Large A".
//
// Reference: hidft.py:135-185 (hidft), hidft.py:160-167 (butterfly).

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "sfft_kernels.cuh"

namespace sfft {

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

// ------------------------------------------ three-pass split (tri) ---
//
// The two-pass back block holds fixed LOW slot bits, but the ascending-J
// output follows the TOP slot bits, so its stores scatter (~9 line requests
// per 16 results on config 5).  Three passes put the last stages in a pass
// whose unit varies only the top 4 slot bits:
//
//  slot a = (b << (S-4)) | (m << F) | x':  x' = low F bits (front), m = MID
//  bits (middle), b = top 4 bits (final).  Sorted position u holds slot
//  brev_S(u); the front's partner index x is the top F sorted bits
//  (x' = brev_F(x)) and its thread position p the low S-F sorted bits
//  (m = brev_MID(p >> 4), b = brev_4(p & 15)).
//
//  front (k_tri_front): loads as k_split_front (coalesced runs of the
//    pattern), runs stages 1..F in registers, transposes through shared
//    memory and writes scratch1[row][p & 15][tri_pos(m, x')]: runs of >= 16
//    consecutive values.
//  middle (k_tri_mid): unit (row, b) = the contiguous block
//    scratch1[row][brev_4(b)] (2^(S-4) values, loaded coalesced straight into
//    registers in its pass-0 layout); runs stages F+1..S-4 (2^F
//    independent transforms over m, twiddles staged once per CTA) and writes
//    scratch2[row][b][pi] with q = perm[pi] (perm: plan->d_tri_perm).
//  final (k_tri_final): a thread owns one pi for all rows of its CTA: its 15
//    twiddles and 16 output positions live in registers; per row it reads
//    scratch2[row][0..15][pi] (coalesced), runs the last 4 stages and stores
//    value b at inv[(b << (S-4)) | q] -- consecutive pi are consecutive
//    outputs when the top 4 pivots are the top bits of j.
// L2-only scratch loads (.cg), last-use loads (.cs) and streaming stores (.cs)
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
__device__ __forceinline__ Cx<float> ld_cs(const Cx<float>* p) {
  Cx<float> r;
  asm volatile("ld.global.cs.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ Cx<double> ld_cs(const Cx<double>* p) {
  Cx<double> r;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs(Cx<float>* p, Cx<float> v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cs(Cx<double>* p, Cx<double> v) {
  asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" :: "l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// streaming store of v at base[i] when i >= 0 (predicated, no branch)
__device__ __forceinline__ void st_cs_if(Cx<float>* base, int32_t i, Cx<float> v) {
  asm volatile("{ .reg .pred q; setp.ge.s32 q, %1, 0; @q st.global.cs.v2.f32 [%0], {%2, %3}; }"
               :: "l"(base + i), "r"(i), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void st_cs_if(Cx<double>* base, int32_t i, Cx<double> v) {
  asm volatile("{ .reg .pred q; setp.ge.s32 q, %1, 0; @q st.global.cs.v2.f64 [%0], {%2, %3}; }"
               :: "l"(base + i), "r"(i), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr(sdst)), "l"(g) : "memory");
}

// Programmatic dependent launch (pdl_wait / pdl_release, sfft_kernels.cuh):
// each tri kernel reads only read-only inputs (signals, plan tables) before
// the wait and releases its dependents only after it, so by induction every
// earlier kernel in the stream has completed once a kernel passes its wait.

#ifndef SFFT_TRI_PF  // front: units prefetched into L2 beyond the one in registers (config 5: 0 -> 145 us, 1 -> 153 us;
                     // loading the next unit after this one's stages instead of before, at
                     // 2 / 3 / 4 CTAs per SM: 149 / 153 / 161 us)
#define SFFT_TRI_PF 0
#endif
#ifndef SFFT_TRI_FRONT_MINB
#define SFFT_TRI_FRONT_MINB 2
#endif
#ifndef SFFT_TRI_FRONT_MINB_D  // complex128
#define SFFT_TRI_FRONT_MINB_D 1
#endif
#ifndef SFFT_TRI_FINAL_MINB_D  // config 6: 2 / 3 / 4 CTAs per SM -> 37.7 / 39.8 / 41.0 us (front: 1 / 2 -> 39.8 / 45.5 us)
#define SFFT_TRI_FINAL_MINB_D 2
#endif
template <typename T, int S, int F>
struct TriGeo {
  static constexpr int L = 4, EXL = 1 << L;   // final: top L slot bits
  static constexpr int MID = S - F - L;        // middle: slot bits [F, F + MID)
  static constexpr int SQ = S - L, NQ = 1 << SQ;
  static constexpr int EX = 1 << F;
  // front
  static constexpr int SP = S - F, NT1 = 256, NSEG = (1 << SP) / NT1, NH = NT1 >> L;
  static constexpr size_t SMEM1 = (size_t)EX * EXL * NH * sizeof(Cx<T>);
  // middle
  static constexpr int E2 = EMax<T>::v < (1 << MID) ? EMax<T>::v : (1 << MID);
  static constexpr int LE2 = ilog2c(E2), NT2 = NQ / E2;
  static constexpr int NPASS2 = (MID + LE2 - 1) / LE2;
  static constexpr int NTW2 = NQ - EX;  // stage-major twiddles of stages F+1 .. S-L
  static constexpr size_t SMEM2 = (size_t)NQ * sizeof(Cx<T>) + (size_t)NTW2 * sizeof(Cx<T>) + (size_t)NQ * 4 * 2;
  // final
  static constexpr int NT3 = 128, NQB = NQ / NT3;
#ifndef SFFT_TRI_FINAL_MINB
#define SFFT_TRI_FINAL_MINB 5
#endif
  static constexpr int MINB3 = sizeof(T) == 4 ? SFFT_TRI_FINAL_MINB : SFFT_TRI_FINAL_MINB_D;
  static_assert(MID >= LE2 && NT1 % EXL == 0 && NQ % NT3 == 0, "tri geometry");
};

// Position of local slot l = (m << F) | x' inside a middle block: the middle
// pass-0 register bits (m mod E2) on top, so thread tid = ((m >> LE2) << F) | x'
// loads register x from position x * NT2 + tid (coalesced, straight into
// registers).
template <typename T, int S, int F>
__device__ __forceinline__ int tri_pos(int m, int xa) {
  using TG = TriGeo<T, S, F>;
  return ((m & (TG::E2 - 1)) << (TG::SQ - TG::LE2)) | ((m >> TG::LE2) << F) | xa;
}

// Front: one CTA per (row, 256 consecutive sorted positions p).  After its
// F stages a thread holds the values of slots (brev_MID(p >> 4) << F |
// brev_F(x)) of middle block p & 15 for all x; the CTA's values of one block
// form runs of >= 16 consecutive positions, written through a staging area
// [p & 15][x][p >> 4 (local)] whose column is XOR-swizzled by (p & 15) ^ x
// (conflict-free for both the per-x writes and the per-block reads).
// twiddles of stages 1..F, passed by value: uniform over the grid, so the
// butterflies take them straight from the constant bank
template <typename T> struct FrontTw { Cx<T> w[15]; };

template <typename T, int S, int F>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? SFFT_TRI_FRONT_MINB : SFFT_TRI_FRONT_MINB_D) k_tri_front(const PlanArgs args, const FrontTw<T> ftw,
                                                                        Cx<T>* __restrict__ scratch, int64_t row0,
                                                                        int64_t nrows) {
  using TG = TriGeo<T, S, F>;
  constexpr int SP = TG::SP, EX = TG::EX, L = TG::L, EXL = TG::EXL, NH = TG::NH, MID = TG::MID, SQ = TG::SQ;
  static_assert(NH == 16, "front staging assumes 16 local p_hi values");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* st = reinterpret_cast<Cx<T>*>(smem_raw);
  // slot bit i -> sample stride (hidft.py:155-158), or the pre-gathered layouts
  auto dstride = [&](int i) -> uint32_t {
    return args.identity == 1   ? (1u << i)
           : args.identity == 2 ? (1u << (S - 1 - i))
                                : (1u << (args.M - 1 - args.used[i]));
  };
  const uint32_t nmask = args.identity ? (uint32_t)((1u << S) - 1u)
                                       : ((args.M >= 32) ? 0xffffffffu : ((1u << args.M) - 1u));
  const int64_t units = nrows * TG::NSEG;
  // sorted bit j <-> slot bit S-1-j: the thread's low 8 position bits are
  // fixed, the CTA-uniform high bits change per unit, partners x add slot
  // bits 0..F-1
  constexpr int TB = 8;  // log2(NT1)
  uint32_t off_t = 0;
#pragma unroll
  for (int j = 0; j < TB; ++j)
    if ((threadIdx.x >> j) & 1u) off_t += dstride(S - 1 - j);
  uint32_t dx[F];
#pragma unroll
  for (int j = 0; j < F; ++j) dx[j] = dstride(F - 1 - j);
  Cx<T> nx[EX];
  // sample address of partner x of unit u (pf: L2 prefetch instead of a load)
  auto unit_off = [&](int64_t u, int64_t& base) {
    const int64_t r = row0 + u / TG::NSEG;
    const uint32_t p0 = (uint32_t)(u % TG::NSEG) * TG::NT1;
#ifdef SFFT_TRI_FOOTPRINT  // timing probe only: every row reads one of two signals
    base = (r & 1) * args.ld;
#else
    base = (args.nshift == 1 ? r : r / args.nshift) * args.ld;
#endif
    const uint32_t rsh = args.nshift == 1 ? 0u : (uint32_t)(r % args.nshift);
    uint32_t off = off_t + (args.identity ? 0u : ((args.negshift - rsh) & nmask));
    for (int j = TB; j < SP; ++j)
      if ((p0 >> j) & 1u) off += dstride(S - 1 - j);
    return off;
  };
  auto fetch = [&](int64_t u) {
    int64_t base;
    const uint32_t off = unit_off(u, base);
#pragma unroll
    for (int x = 0; x < EX; ++x) {
      uint32_t o = off;
#pragma unroll
      for (int j = 0; j < F; ++j)
        if ((x >> j) & 1) o += dx[j];
      if (sizeof(T) == 8 && args.in_c64) {
        const Cx<float> sv = load_sample(reinterpret_cast<const Cx<float>*>(args.sig) + base + (o & nmask));
        nx[x] = Cx<T>{(T)sv.x, (T)sv.y};
      } else {
        nx[x] = load_sample(reinterpret_cast<const Cx<T>*>(args.sig) + base + (o & nmask));
      }
    }
  };
  auto prefetch = [&](int64_t u) {
    int64_t base;
    const uint32_t off = unit_off(u, base);
    const size_t esz_in = (sizeof(T) == 8 && args.in_c64) ? sizeof(Cx<float>) : sizeof(Cx<T>);
    const char* sig = reinterpret_cast<const char*>(args.sig);
#pragma unroll
    for (int x = 0; x < EX; ++x) {
      uint32_t o = off;
#pragma unroll
      for (int j = 0; j < F; ++j)
        if ((x >> j) & 1) o += dx[j];
      asm volatile("prefetch.global.L2 [%0];" :: "l"(sig + (base + (o & nmask)) * esz_in));
    }
  };
  int64_t u = blockIdx.x;
  if (u < units) fetch(u);  // signals are read-only here
#pragma unroll
  for (int k = 2; k < 2 + SFFT_TRI_PF; ++k)
    if (u + k * gridDim.x < units) prefetch(u + k * gridDim.x);
  pdl_wait();               // scratch1 is free (the previous chunk's middle pass completed)
  pdl_release();
  for (; u < units; u += gridDim.x) {
    Cx<T> v[EX];
#pragma unroll
    for (int x = 0; x < EX; ++x) v[x] = nx[x];
    if (u + gridDim.x < units) fetch(u + gridDim.x);
    if (SFFT_TRI_PF > 0 && u + (1 + SFFT_TRI_PF) * gridDim.x < units) prefetch(u + (1 + SFFT_TRI_PF) * gridDim.x);
#pragma unroll
    for (int k = 1; k <= F; ++k) {  // stage k pairs slot bit k-1 = x bit F-k (hidft.py:160-167)
      const int lb = F - k;
#pragma unroll
      for (int x = 0; x < EX; ++x) {
        if (x & (1 << lb)) continue;
        const uint32_t h = brev_c<F>((uint32_t)x) & ((1u << (k - 1)) - 1u);
        bfly(v[x], v[x | (1 << lb)], ftw.w[(1 << (k - 1)) - 1 + h]);
      }
    }
    {
      const int lo = threadIdx.x & (EXL - 1), hl = threadIdx.x >> L;
#pragma unroll
      for (int x = 0; x < EX; ++x) st[(lo * EX + x) * NH + (hl ^ ((lo ^ x) & (NH - 1)))] = v[x];
    }
    __syncthreads();
    // block lo gets slots m = brev_MID(ph0 + hl) = m0 | brev_4(hl) << (MID - 4)
    const uint32_t p0 = (uint32_t)(u % TG::NSEG) * TG::NT1;
    const uint32_t m0 = brev_c<MID>(p0 >> L);
    Cx<T>* rowbase = scratch + ((u / TG::NSEG) << S);
#pragma unroll
    for (int n = 0; n < EX; ++n) {
      const int id = n * TG::NT1 + threadIdx.x;
      const int xa = id & (EX - 1), hb = (id >> F) & (NH - 1), lo = id >> (F + 4);
      const int hl = (int)brev_c<4>((uint32_t)hb), x = (int)brev_c<F>((uint32_t)xa);
      const int m = (int)(m0 | ((uint32_t)hb << (MID - 4)));
      rowbase[((int64_t)lo << SQ) + tri_pos<T, S, F>(m, xa)] = st[(lo * EX + x) * NH + (hl ^ ((lo ^ x) & (NH - 1)))];
    }
    __syncthreads();  // st is rewritten by the next unit
  }
}

// Middle: persistent over units (row, b); the next unit's block is loaded into
// registers (pass-0 layout) while this one runs.
template <typename T, int S, int F>
__global__ void __launch_bounds__(TriGeo<T, S, F>::NT2) k_tri_mid(const Cx<T>* __restrict__ scr1,
                                                                  Cx<T>* __restrict__ scr2, int64_t nrows,
                                                                  const Cx<T>* __restrict__ tw,
                                                                  const int32_t* __restrict__ perm,
                                                                  const int32_t* __restrict__ spos,
                                                                  const int32_t* __restrict__ ppos) {
  using TG = TriGeo<T, S, F>;
  constexpr int EX = TG::EX, MID = TG::MID, NQ = TG::NQ, SQ = TG::SQ, L = TG::L, E = TG::E2, LE = TG::LE2,
                NT = TG::NT2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<T>* sd = reinterpret_cast<Cx<T>*>(smem_raw);  // NQ, swizzled local slot l = (m << F) | x'
  Cx<T>* stw = sd + NQ;                             // stage-major twiddles of stages F+1 .. S-L
  int32_t* sperm = reinterpret_cast<int32_t*>(stw + TG::NTW2);  // perm, or ppos with the conflict-free layout
  int32_t* sspos = sperm + NQ;                                  // spos (conflict-free layout only)
  const int tid = threadIdx.x;
  // conflict-free layout (plan->d_tri_spos / d_tri_ppos, sfft_plan.cu): the
  // last pass stores at spos and the epilogue reads pi at ppos[pi]
  const bool cf = spos != nullptr;
  // tables staged asynchronously (cp.async) while the first unit's block loads
  for (int i = tid; i < TG::NTW2; i += NT) cp_async_elem(stw + i, tw + EX - 1 + i);
  for (int i = tid; i < NQ / 4; i += NT) cp_async16(sperm + 4 * i, (cf ? ppos : perm) + 4 * i);
  if (cf)
    for (int i = tid; i < NQ / 4; i += NT) cp_async16(sspos + 4 * i, spos + 4 * i);
  cp_async_commit();
  const int a = tid & (EX - 1), mr = tid >> F;
  const int64_t units = nrows << L;
  Cx<T> nx[E];
  auto fetch = [&](int64_t u) {
    const Cx<T>* src = scr1 + ((u >> L) << S) + ((int64_t)brev_c<L>((uint32_t)(u & (TG::EXL - 1))) << SQ) + tid;
#pragma unroll
    for (int x = 0; x < E; ++x) nx[x] = ld_cg(src + x * NT);
  };
  int64_t u = blockIdx.x;
  pdl_wait();  // scratch1 written by this chunk's front pass
  pdl_release();
  if (u < units) fetch(u);
  cp_async_wait<0>();
  __syncthreads();  // staged tables
  for (; u < units; u += gridDim.x) {
    Cx<T> v[E];
#pragma unroll
    for (int x = 0; x < E; ++x) v[x] = nx[x];
    if (u + gridDim.x < units) fetch(u + gridDim.x);
#pragma unroll
    for (int ps = 0; ps < TG::NPASS2; ++ps) {
      const int w0 = pass_w0(ps, MID, LE);
      if (ps > 0) {
#pragma unroll
        for (int x = 0; x < E; ++x) v[x] = sd[swz<T, SQ>((slot_of<MID, LE>(ps, mr, x) << F) | a)];
      }
      const int b0 = ps * LE, b1 = (b0 + LE < MID) ? b0 + LE : MID;
#pragma unroll
      for (int beta = b0; beta < b1; ++beta) {  // global stage F + beta + 1 pairs m bit beta
        const int lb = beta - w0;
#pragma unroll
        for (int x = 0; x < E; ++x) {
          if (x & (1 << lb)) continue;
          const int m = slot_of<MID, LE>(ps, mr, x);
          const int h = a | ((m & ((1 << beta) - 1)) << F);
          bfly(v[x], v[x | (1 << lb)], stw[(1 << (F + beta)) - EX + h]);
        }
      }
      if (cf && ps == TG::NPASS2 - 1) {
        if (ps > 0) __syncthreads();  // every thread has read this pass's inputs from sd
#pragma unroll
        for (int x = 0; x < E; ++x) sd[sspos[x * NT + tid]] = v[x];
      } else {
#pragma unroll
        for (int x = 0; x < E; ++x) sd[swz<T, SQ>((slot_of<MID, LE>(ps, mr, x) << F) | a)] = v[x];
      }
      __syncthreads();
    }
    Cx<T>* dst = scr2 + ((u >> L) << S) + ((u & (TG::EXL - 1)) << SQ);
#pragma unroll
    for (int n = 0; n < E; ++n) {
      const int pi = tid + n * NT;
      dst[pi] = cf ? sd[sperm[pi]] : sd[swz<T, SQ>(sperm[pi])];
    }
    __syncthreads();  // sd is rewritten by the next unit
  }
}

// Final: a thread owns position pi for the rows of its CTA (twiddles and
// output positions in registers); the next row is prefetched.
template <typename T, int S, int F>
__global__ void __launch_bounds__(TriGeo<T, S, F>::NT3, TriGeo<T, S, F>::MINB3) k_tri_final(const PlanArgs args, const Cx<T>* __restrict__ scr2,
                                                                    int64_t row0, int64_t nrows, int nper,
                                                                    const Cx<T>* __restrict__ twf,
                                                                    const int32_t* __restrict__ invf,
                                                                    const int32_t* __restrict__ perm) {
  using TG = TriGeo<T, S, F>;
  constexpr int NQ = TG::NQ, SQ = TG::SQ, EXL = TG::EXL, L = TG::L;
  __shared__ Cx<T> sw[EXL - 1][TG::NT3];  // this CTA's pi block: twiddles of the last L stages
  const int qb = blockIdx.x % TG::NQB;
  const int64_t first = blockIdx.x / TG::NQB;
  if (first >= nrows) return;
  const int pi = qb * TG::NT3 + threadIdx.x;
  Cx<T> nx[EXL];
  auto fetch = [&](int64_t rr) {
    const Cx<T>* src = scr2 + (rr << S) + pi;
#pragma unroll
    for (int b = 0; b < EXL; ++b) nx[b] = ld_cs(src + ((int64_t)b << SQ));
  };
  const int q = perm[pi];
#pragma unroll
  for (int j = 0; j < EXL - 1; ++j) sw[j][threadIdx.x] = twf[(int64_t)j * NQ + pi];  // read by this thread only
  int32_t e[EXL];
#pragma unroll
  for (int b = 0; b < EXL; ++b) e[b] = invf ? invf[(int64_t)b * NQ + pi] : ((b << SQ) | q);
  pdl_wait();  // scratch2 written by this chunk's middle pass
  pdl_release();
  fetch(first);
  const T scale = (T)args.scale1;
  for (int64_t rr = first; rr < nrows; rr += nper) {
    Cx<T> v[EXL];
#pragma unroll
    for (int b = 0; b < EXL; ++b) v[b] = nx[b];
    if (rr + nper < nrows) fetch(rr + nper);
#pragma unroll
    for (int t = 0; t < L; ++t) {  // global stage SQ + t + 1 pairs slot bit SQ + t = b bit t
#pragma unroll
      for (int b = 0; b < EXL; ++b) {
        if (b & (1 << t)) continue;
        bfly(v[b], v[b | (1 << t)], sw[(1 << t) - 1 + (b & ((1 << t) - 1))][threadIdx.x]);
      }
    }
    const int64_t r = row0 + rr;
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + r * args.ld1;
#pragma unroll
    for (int b = 0; b < EXL; ++b) st_cs_if(o1, e[b], cscale(v[b], scale));
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + r * args.ld2;
#pragma unroll
      for (int b = 0; b < EXL; ++b) o2[(b << SQ) | q] = v[b];
    }
  }
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
  {
    // legal while a stream captures once this thread's capture mode is relaxed
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    SFFT_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
    const cudaError_t e = cudaMemPoolCreate(&p, &props);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (e != cudaSuccess) return cuda_fail(e, "scratch pool creation");
  }
  uint64_t keep = ~0ull;
  SFFT_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
  pools[dev] = p;
  *pool = p;
  return SFFT_OK;
}

// Scratch of the three-pass split, kept per (device, stream) and reused by
// every call on that stream: calls on one stream are ordered, and a pass
// writes scratch only after its predecessor (hence the previous call) has
// completed.  Allocating per call from a stream-ordered pool instead puts a
// memory node into every captured graph, and alternating between graphs
// that hold such nodes costs the driver a remap of the memory at each switch
// (config 5 in bench.py: 137 us per step with one graph, 173-362 us when a
// 32-step graph alternates with tail graphs).  A graph keeps the buffer of
// the stream it was captured on: replay it on one stream at a time.  Up to
// kStreamScratch streams per device keep a buffer; further streams fall back
// to the pool (allocated and freed per call).
constexpr int kStreamScratch = 8;
struct StreamScratch {
  cudaStream_t stream;
  void* ptr;
  size_t bytes;
};
static std::mutex g_ss_mu;
static std::map<int, std::vector<StreamScratch>> g_ss;
static std::vector<void*> g_ss_retired;  // outgrown buffers, kept until process exit

// *ptr: scratch of at least `bytes` for stream st; *pooled: the caller frees it (cudaFreeAsync)
static int stream_scratch(int dev, cudaStream_t st, size_t bytes, void** ptr, bool* pooled) {
  *pooled = false;
  {
    std::lock_guard<std::mutex> lk(g_ss_mu);
    auto& v = g_ss[dev];
    bool listed = false;
    for (auto& e : v) {
      if (e.stream != st) continue;
      listed = true;
      if (e.bytes < bytes) {
        // the old buffer is retired, not freed: a CUDA graph captured
        // earlier on this stream may still reference it; the
        // plain allocation is legal inside a capture with the thread's
        // capture mode relaxed (as below)
        void* np = nullptr;
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        SFFT_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
        const cudaError_t ge = cudaMalloc(&np, bytes);
        cudaThreadExchangeStreamCaptureMode(&mode);
        if (ge != cudaSuccess) return cuda_fail(ge, "stream scratch allocation");
        g_ss_retired.push_back(e.ptr);
        e.ptr = np;
        e.bytes = bytes;
      }
      *ptr = e.ptr;
      return SFFT_OK;
    }
    if (!listed && (int)v.size() < kStreamScratch) {
      // a plain allocation is legal while a stream captures once this
      // thread's capture mode is relaxed (as PyTorch's allocator does)
      cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
      SFFT_CUDA(cudaThreadExchangeStreamCaptureMode(&mode));
      void* p = nullptr;
      const cudaError_t e = cudaMalloc(&p, bytes);
      cudaThreadExchangeStreamCaptureMode(&mode);
      if (e != cudaSuccess) return cuda_fail(e, "stream scratch allocation");
      v.push_back({st, p, bytes});
      *ptr = p;
      return SFFT_OK;
    }
  }
  cudaMemPool_t pool;
  if (int rc = scratch_pool(dev, &pool)) return rc;
  SFFT_CUDA(cudaMallocFromPoolAsync(ptr, bytes, pool, st));
  *pooled = true;
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

// kernel launches run_split issues for `rows` rows (sfft_launch_count)
template <typename T, int S, int LC>
static int split_launches(int64_t rows, int64_t* n) {
  using SG = SplitGeo<T, S, LC>;
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

// cudaLaunchKernelEx, optionally as a programmatic dependent launch
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                            bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// rows per chunk of the three-pass split: each of the two scratch buffers
// up to SFFT_TRI_SCRATCH_MB (default 64 MiB: 2 chunks of 128 rows on config
// 5; measured 16/24/32/48/64/96/128 MiB -> 166/153/144/141/140/144/146 us)
static int64_t tri_chunk_rows(int64_t rows, size_t row_bytes) {
  static const int64_t scr_mb = [] {
    const char* e = getenv("SFFT_TRI_SCRATCH_MB");
    return (int64_t)(e ? std::max(1, atoi(e)) : 64);
  }();
  return std::max<int64_t>(1, std::min<int64_t>(rows, (scr_mb << 20) / (int64_t)row_bytes));
}

template <typename T, int S, int F>
static int tri_launches(int64_t rows, int64_t* n) {
  const int64_t chunk = tri_chunk_rows(rows, sizeof(Cx<T>) << S);
  *n = rows > 0 ? 3 * ((rows + chunk - 1) / chunk) : 0;
  return SFFT_OK;
}

template <typename T, int S, int F>
static int run_tri(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  using TG = TriGeo<T, S, F>;
  if (!p->d_tri_perm) return fail(SFFT_ERR_INVALID, "plan has no three-pass tables");
  const int32_t* invf = inv1 == p->d_inv_elem ? p->d_tri_inv_elem
                        : inv1 == p->d_inv_node ? p->d_tri_inv_node
                                                : nullptr;
  if (inv1 && !invf) return fail(SFFT_ERR_INVALID, "no final-pass map for this output");
  auto front = k_tri_front<T, S, F>;
  auto mid = k_tri_mid<T, S, F>;
  auto fin = k_tri_final<T, S, F>;
  int occ1 = 0, occ2 = 0, occ3 = 0, rc;
  if ((rc = kernel_occupancy(front, TG::NT1, TG::SMEM1, &occ1))) return rc;
  if ((rc = kernel_occupancy(mid, TG::NT2, TG::SMEM2, &occ2))) return rc;
  if ((rc = kernel_occupancy(fin, TG::NT3, 0, &occ3))) return rc;
  const int64_t rows = a.B * a.nshift;
  if (rows == 0) return SFFT_OK;
  const size_t row_bytes = sizeof(Cx<T>) << S;
  const int64_t chunk = tri_chunk_rows(rows, row_bytes);
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  void* scr = nullptr;
  bool pooled = false;
  if ((rc = stream_scratch(dev, st, 2 * (size_t)chunk * row_bytes, &scr, &pooled))) return rc;
  Cx<T>* s1 = (Cx<T>*)scr;
  Cx<T>* s2 = s1 + ((size_t)chunk << S);
  const Cx<T>* tw = reinterpret_cast<const Cx<T>*>(p->d_twiddles);
  const Cx<T>* twf = reinterpret_cast<const Cx<T>*>(p->d_tri_tw);
  const int64_t sms = num_sms();
  FrontTw<T> ftw;
  std::memcpy(&ftw, p->tri_front_tw, sizeof(Cx<T>) * std::min<int64_t>(15, p->A - 1));
  static const bool pdl = [] {
    const char* e = getenv("SFFT_TRI_PDL");
    return !(e && atoi(e) == 0);
  }();
  // the call's first front joins the stream's PDL chain (sfft_hidft.cu,
  // pdl_join) when its signals do not overlap the chain's outputs: its
  // pre-wait loads read only the signals, so it gathers while the previous
  // call's final pass drains (scratch is written only after its wait)
  const size_t esz_in = (sizeof(T) == 8 && a.in_c64) ? 8 : sizeof(Cx<T>);
  const ByteRange in[1] = {{(uintptr_t)a.sig, (uintptr_t)a.sig + (size_t)((a.B - 1) * a.ld +
                                                   (a.identity ? (1ll << S) : (1ll << a.M))) * esz_in}};
  const ByteRange outs[2] = {
      {(uintptr_t)a.out1, (uintptr_t)a.out1 + (size_t)((rows - 1) * a.ld1 + a.n1) * sizeof(Cx<T>)},
      {(uintptr_t)a.out2, a.out2 ? (uintptr_t)a.out2 + (size_t)((rows - 1) * a.ld2 + (1ll << S)) * sizeof(Cx<T>)
                                 : 0}};
  const bool pdl_first = pdl_join(st, in, 1, outs, 2, pdl && !pooled && a.identity == 0);
  cudaError_t e = cudaSuccess;
  for (int64_t r0 = 0; r0 < rows && e == cudaSuccess; r0 += chunk) {
    const int64_t n = std::min(chunk, rows - r0);
    const int64_t g1 = std::min<int64_t>(n * TG::NSEG, sms * occ1);
    e = launch_k(front, (unsigned)g1, TG::NT1, TG::SMEM1, st, pdl && (r0 > 0 || pdl_first), a, ftw, s1, r0, n);
    const int64_t g2 = std::min<int64_t>(n << TG::L, sms * occ2);
    if (e == cudaSuccess)
      e = launch_k(mid, (unsigned)g2, TG::NT2, TG::SMEM2, st, pdl, (const Cx<T>*)s1, s2, n, tw,
                   (const int32_t*)p->d_tri_perm, (const int32_t*)p->d_tri_spos, (const int32_t*)p->d_tri_ppos);
    const int nper = (int)std::max<int64_t>(1, std::min<int64_t>(n, sms * occ3 / TG::NQB));
    if (e == cudaSuccess)
      e = launch_k(fin, (unsigned)(nper * TG::NQB), TG::NT3, 0, st, pdl, a, (const Cx<T>*)s2, r0, n, nper, twf,
                   invf, (const int32_t*)p->d_tri_perm);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (pooled) cudaFreeAsync(scr, st);
  if (e != cudaSuccess) return cuda_fail(e, "three-pass transform launch");
  return SFFT_OK;
}

// SFFT_SPLIT_PASSES=2 selects the two-pass split (A/B measurements)
static bool use_tri() {
  static const bool v = [] {
    const char* e = getenv("SFFT_SPLIT_PASSES");
    return !(e && atoi(e) == 2);
  }();
  return v;
}

// ------------------------------------------ TMA head + final (two-pass) ---
//
// The three-pass split reads whole 128 B lines in its front pass and needs a
// middle pass (a second L2 round trip) because the first 12 stages run
// across the lines of the pattern.  The head pass does the front's and the
// middle's work in one kernel: slot a = (b << SQ) | q, and when the two
// smallest sample strides are 1 and 2 (config 5: pivots M-1, M-2 present)
// the 16 values of a q sit in one 128 B line, b's low-offset bits in the
// line's low positions.  A CTA owns a unit (row, c): the P values of every
// line at offset off_c (P = 2: 16 B, 8 units per row; P = 4: 32 B, 4 units),
// i.e. P independent 2^SQ-slot transforms over q.  Its samples are fetched
// by TMA: the q bits of the pattern form runs of consecutive strides, the
// three longest runs become dims 1-3 of a rank-5 tensor map over the signal
// batch (dim 0 = the P-element piece, dim 4 = the row) and the remaining q
// bits are enumerated by one cp.async.bulk.tensor per combination, so the
// LSU never issues a gather instruction.  The landing layout is a bit
// permutation of q (HeadTma::qw); pass 0 reads it into registers, runs
// stages 1-4 and continues with the swizzled single-CTA layout for stages
// 5..SQ; the last pass stores each value at its final-pass position pi and
// the b value's block leaves for scratch[row][b][pi] by one bulk copy (pi:
// the final pass's output order).  The final pass is k_fin3 (tensor loads
// and stores) for blocked output maps, else k_fin2 (k_tri_final's scheme
// with FFMA2 and register twiddles).  Every stream of the path carries an L2
// eviction priority so that the scratch chunk stays in L2 between the two
// kernels.  Reference: hidft.py:34-49 (gather), 160-167.
struct HeadTma {
  int nops, nleft, P;
  uint32_t left_d[16];  // element offset of each enumerated (leftover) q bit
  uint32_t k1, k2, k3;  // dim j covers element-offset bits [k_j, k_j+1) of the row (dim 0: [0, k1))
  uint32_t qw[16];      // landing-layout weight of q bit i (in q units)
  uint32_t dfix[4];     // element offset of b bit 0..3 (slot bits SQ..SQ+3)
  int len[3];
  uint8_t tq[16];       // pass-0 thread bit i -> q bit tq[i] (q bits LE.., ascending landing weight)
};

template <typename T, int S, int P>
struct HeadGeo {
  static constexpr int L = 4, SQ = S - L, NQ = 1 << SQ, NC = 16 / P;
  static constexpr int E = 16, LE = 4;       // slots per thread, one b value per thread
  static constexpr int TPB = NQ / E;         // threads per b value
  static constexpr int NT = P * TPB;         // transform threads
  static constexpr int NTT = NT + 32;        // + one warp that issues the tensor copies
  static constexpr int NPASS = (SQ + LE - 1) / LE;
  static constexpr int NTW = NQ - 16;        // stage-major twiddles 15 .. NQ-2 (stages 5 .. SQ)
  // NL landing buffers (TMA) + working buffer (swizzled slots) + twiddles + 2 NL mbarriers
#ifndef SFFT_HEAD_NL  // landing buffers (config 5 with the bulk epilogue and per-b-value groups: 1 -> 120.6 us, 2 -> 116.2 us per step)
#define SFFT_HEAD_NL 2
#endif
  static constexpr int NL = P == 2 ? SFFT_HEAD_NL : 1;
  static constexpr size_t SMEM = (NL + 1) * (size_t)P * NQ * sizeof(Cx<T>) + (size_t)NTW * sizeof(Cx<T>) + 16 * NL;
  static_assert(sizeof(T) == 4 && SQ >= 2 * LE && E <= TPB, "head pass: complex64, at least 2 register passes");
};

// L2 eviction priorities of the head path's four streams (each -D...=0/1;
// config 5, one box, 256-row step): none 110.3 us; signal copies, scratch
// loads and output stores evict_first 100.4-101.4 us; the same with the
// scratch copies evict_last 104.0 us; without the output hint 105.7-106.3 us;
// signal / scratch-load hint alone 103.2 / 105.4 us.  Everything that is
// read or written once leaves L2 first, and the scratch (default priority)
// survives from the head pass to the final pass.
#ifndef SFFT_SIG_HINT  // evict_first on the head pass's signal copies
#define SFFT_SIG_HINT 1
#endif
#ifndef SFFT_FIN_LOAD_HINT  // evict_first on the final pass's scratch loads (k_fin3)
#define SFFT_FIN_LOAD_HINT 1
#endif
#ifndef SFFT_SCR_HINT  // evict_last on the head pass's scratch copies
#define SFFT_SCR_HINT 0
#endif
#ifndef SFFT_OUT_HINT  // evict_first on the final pass's output stores
#define SFFT_OUT_HINT 1
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// twiddles of stages 1..4 and their rotations i*w (uniform over the grid)
struct FrontTw2 { Cx<float> w[15], iw[15]; };

__device__ __forceinline__ void mbar_init(uint32_t a, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(a) : "memory");
}
// SFFT_TIMELINE=1 (host env): per launch of the head path's kernels, the
// first CTA start, the first CTA past griddepcontrol.wait and the last CTA
// end (globaltimer, ns) are recorded and printed at exit (stderr) -- a
// device-side timeline of the pipeline (probe only; tl == nullptr otherwise)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tl_mark(unsigned long long* tl, int what) {
  if (tl && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (what == 2) atomicMax(tl + 2, t);
    else atomicMin(tl + what, t);
  }
}

// -DSFFT_HEAD_CLK: per-phase cycle counts of CTA 0 (warps 0 and NT/32-1), printed
// at kernel exit (probe only)
#ifdef SFFT_HEAD_CLK
#define HCLK(i) do { const long long t__ = clock64(); hacc[i] += t__ - hlast; hlast = t__; } while (0)
#else
#define HCLK(i) do { } while (0)
#endif

// barrier among the NT transform threads only (the copy warp runs its own loop)
template <int NT>
__device__ __forceinline__ void work_sync() { asm volatile("bar.sync 1, %0;" :: "n"(NT) : "memory"); }
// barrier among the warps of one b value's group (named barrier 2 + group);
// SFFT_HEAD_GROUPS=0: one barrier over all transform threads.  With the
// register epilogue the groups made no difference (126.1-126.4 against 126.5
// us per config-5 step); with the bulk epilogue and two landing buffers
// nothing couples the two b values of a unit any more and the groups' FMA
// and shared-memory phases interleave (120.4 -> 116.3 us)
#ifndef SFFT_HEAD_GROUPS
#define SFFT_HEAD_GROUPS 1
#endif
#if SFFT_HEAD_GROUPS
#define HEAD_SYNC() group_sync<NTG>(bl)
#else
#define HEAD_SYNC() work_sync<NT>()
#endif
template <int NTG>
__device__ __forceinline__ void group_sync(int grp) { asm volatile("bar.sync %0, %1;" :: "r"(2 + grp), "n"(NTG) : "memory"); }

// Persistent: CTA i serves units i, i + grid, ...; a copy warp fills the
// landing buffer with unit u+1 (tensor copies; it alone stalls when the TMA
// queue is full) as soon as the transform threads have read unit u from it,
// so the copies run while unit u is transformed in the working buffer.
// Persistent: CTA i serves units i, i + grid, ...; a copy warp fills NL
// landing buffers with the next units (tensor copies; it alone stalls when
// the TMA queue is full) as soon as the transform threads have read the
// buffer's previous unit, so the copies of units u+1 and u+2 run while unit
// u is transformed in the working buffer.
template <typename T, int S, int P>
__global__ void __launch_bounds__(HeadGeo<T, S, P>::NTT, 1)
k_head(const __grid_constant__ CUtensorMap tm, const HeadTma ht, const FrontTw2 ftw, const Cx<T>* __restrict__ tw,
       const int32_t* __restrict__ perm, Cx<T>* __restrict__ scratch, int64_t row0, int64_t units,
       const int32_t* __restrict__ cf_spos, const int32_t* __restrict__ cf_ppos, int bulk,
       unsigned long long* tl) {
  tl_mark(tl, 0);
  using HG = HeadGeo<T, S, P>;
  constexpr int SQ = HG::SQ, NQ = HG::NQ, E = HG::E, LE = HG::LE, TPB = HG::TPB, NT = HG::NT, NC = HG::NC;
  constexpr int LP = P == 4 ? 2 : 1;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NL = HG::NL;
  [[maybe_unused]] constexpr int NTG = NT / P;
  Cx<T>* land = reinterpret_cast<Cx<T>*>(smem_raw);  // NL x P x NQ, TMA box order
  Cx<T>* work = land + NL * P * NQ;                  // P x NQ, swizzled slots per b value
  Cx<T>* stw = work + P * NQ;                        // twiddles of stages 5 .. SQ
  const uint32_t full0 = smem_addr(stw + HG::NTW), empty0 = full0 + 8 * NL;  // full[NL], empty[NL]
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < NL; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid >= NT) {  // copy warp (signals are read-only: the first copies may overlap the previous kernel)
    const int lane = tid - NT;
    const int box = (NQ / ht.nops) * P;
    uint32_t it = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
      const int lb = it % NL;
      const uint32_t full = full0 + 8 * lb;
      Cx<T>* lbuf = land + lb * P * NQ;
      // landing buffer lb is free once the transform threads read unit it - NL from it
      if (it >= (uint32_t)NL) mbar_wait(empty0 + 8 * lb, ((it - NL) / NL) & 1);
#if defined(SFFT_HEAD_PROBE) && SFFT_HEAD_PROBE == 2  // timing probe: copies of the first units only
      if (it >= (uint32_t)NL) {
        if (lane == 0) mbar_arrive(full);
        continue;
      }
#endif
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(full), "r"((uint32_t)(P * NQ * sizeof(Cx<T>))) : "memory");
      }
      __syncwarp();
      const int64_t rr = u / NC;
      const int c = (int)(u % NC);
      uint32_t offc = 0;
#pragma unroll
      for (int j = 0; j < 4 - LP; ++j)
        if ((c >> j) & 1) offc += ht.dfix[j];
      for (int o = lane; o < ht.nops; o += 32) {
        uint32_t e = offc;
        for (int j = 0; j < ht.nleft; ++j)
          if ((o >> j) & 1) e += ht.left_d[j];
        const int c0 = (int)(e & ((1u << ht.k1) - 1u));
        const int c1 = (int)((e >> ht.k1) & ((1u << (ht.k2 - ht.k1)) - 1u));
        const int c2 = (int)((e >> ht.k2) & ((1u << (ht.k3 - ht.k2)) - 1u));
        const int c3 = (int)(e >> ht.k3);
        const int c4 = (int)(row0 + rr);
#if SFFT_SIG_HINT
        // probe: signal lines first out of L2 (they are read by the 8 units of a row within a short window)
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;"
            :: "r"(smem_addr(lbuf + (size_t)o * box)), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
               "r"(full), "l"(l2_policy_evict_first()) : "memory");
#else
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :: "r"(smem_addr(lbuf + (size_t)o * box)), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
               "r"(full) : "memory");
#endif
      }
    }
    return;
  }
  // Warp bits 0..LP-1 pick the b value inside the piece: each b value's
  // transform is done by its own group of NT/P threads with its own named
  // barriers, so the groups drift out of phase and overlap each other's
  // shared-memory and FMA phases (as two CTAs would); a half-warp works on
  // one b value, so its 16 lanes hit 16 distinct 8 B word slots in the
  // swizzled passes (conflict-free).  Pass-0 thread bit i holds q bit tq[i]
  // (host order: ascending landing weight).
  for (int i = tid; i < HG::NTW; i += NT) cp_async_elem(stw + i, tw + 15 + i);
  cp_async_commit();
  const int bl = (tid >> 5) & (P - 1), tt = (tid & 31) | ((tid >> (5 + LP)) << 5);
  uint32_t qt = 0, base = 0;
#pragma unroll
  for (int i = 0; i < SQ - LE; ++i)
    if ((tt >> i) & 1) {
      qt |= 1u << ht.tq[i];
      base += ht.qw[ht.tq[i]];
    }
  const int tb0 = swz<T, SQ>((int)qt);
  Cx<T>* sb = work + bl * NQ;
  cp_async_wait<0>();
  work_sync<NT>();  // twiddles staged by all groups
  bool waited = false;
  uint32_t it = 0;
  // the thread that issues (and waits for) the bulk epilogue copies: one per barrier group
  const int issuer = SFFT_HEAD_GROUPS ? bl * 32 : 0;
#if defined(SFFT_HEAD_LAG) && SFFT_HEAD_GROUPS
  // probe: group 1 starts SFFT_HEAD_LAG cycles late, so the two groups' shared-memory
  // and FMA phases interleave instead of running in lockstep
  if (bl == 1) {
    const long long t0 = clock64();
    while (clock64() - t0 < SFFT_HEAD_LAG) { }
  }
#endif
#ifdef SFFT_HEAD_CLK
  long long hacc[12] = {0}, hlast = clock64();
#endif
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    Cx<T> v[E];
    const int lb = it % NL;
    const Cx<T>* lbuf = land + lb * P * NQ;
    HCLK(11);
    mbar_wait(full0 + 8 * lb, (it / NL) & 1);
    HCLK(0);
#pragma unroll
    for (int x = 0; x < E; ++x) {
      uint32_t q = base;
#pragma unroll
      for (int i = 0; i < LE; ++i)
        if ((x >> i) & 1) q += ht.qw[i];
      v[x] = lbuf[q * P + bl];
    }
    // bulk epilogue: the previous unit's stores have read the working buffer
    if (bulk && tid == issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    HEAD_SYNC();  // the group's landing reads and its previous epilogue reads of work done
    HCLK(1);
    if ((tid & 31) == 0) mbar_arrive(empty0 + 8 * lb);
#if defined(SFFT_HEAD_PROBE) && SFFT_HEAD_PROBE == 1  // timing probe: copies and scratch stores only
    if (!waited) {
      pdl_wait();
      pdl_release();
      waited = true;
    }
    {
      const int64_t rr = u / NC;
      const int b = (int)(u % NC) | (LP == 1 ? (bl << 3) : (((bl & 1) << 3) | ((bl >> 1) << 2)));
      Cx<T>* dst = scratch + ((int64_t)rr << S) + ((int64_t)b << SQ) + tt;
#pragma unroll
      for (int n = 0; n < E; ++n) dst[n * TPB] = v[n];
    }
    continue;
#endif
    // stages 1..LE: twiddle index a mod 2^beta = x mod 2^beta, uniform over the grid
#pragma unroll
    for (int beta = 0; beta < LE; ++beta) {
#pragma unroll
      for (int x = 0; x < E; ++x) {
        if (x & (1 << beta)) continue;
        const int j = (1 << beta) - 1 + (x & ((1 << beta) - 1));
        bfly2(v[x], v[x | (1 << beta)], ftw.w[j], ftw.iw[j]);
      }
    }
    HCLK(2);
#pragma unroll
    for (int x = 0; x < E; ++x) sb[tb0 ^ swz<T, SQ>(x)] = v[x];
    HCLK(3);
    HEAD_SYNC();
    HCLK(4);
#pragma unroll
    for (int p = 1; p < HG::NPASS; ++p) {
      const int tb = swz<T, SQ>(slot_t<SQ, LE>(p, tt));
#pragma unroll
      for (int x = 0; x < E; ++x) v[x] = sb[tb ^ swz<T, SQ>(slot_x<SQ, LE>(p, x))];
      const int b0 = p * LE, b1 = (b0 + LE < SQ) ? b0 + LE : SQ, w0 = pass_w0(p, SQ, LE);
#pragma unroll
      for (int beta = b0; beta < b1; ++beta) {
        const int lb = beta - w0;
        // butterflies of this stage share twiddle h = a mod 2^beta: one per value of x's bits below lb
#pragma unroll
        for (int xl = 0; xl < (1 << lb); ++xl) {
          const int a0 = slot_of<SQ, LE>(p, tt, xl);
          const Cx<T> w = stw[(1 << beta) - 16 + (a0 & ((1 << beta) - 1))];
          const Cx<T> iw = rot_i(w);
#pragma unroll
          for (int x = xl; x < E; x += (1 << lb)) {
            if (x & (1 << lb)) continue;
            bfly2(v[x], v[x | (1 << lb)], w, iw);
          }
        }
      }
      HCLK(5);
      if (cf_spos && p == HG::NPASS - 1) {
        // conflict-free layout of the last stores and the epilogue reads
        // (plan->d_head_spos / d_head_ppos, sfft_plan.cu): other positions
        // than this pass read, so every thread must have read its inputs first
        HEAD_SYNC();
#pragma unroll
        for (int x = 0; x < E; ++x) sb[__ldg(cf_spos + x * TPB + tt)] = v[x];
        if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      } else {
#pragma unroll
        for (int x = 0; x < E; ++x) sb[tb ^ swz<T, SQ>(slot_x<SQ, LE>(p, x))] = v[x];  // in place: same positions
      }
      HCLK(6);
      HEAD_SYNC();
      HCLK(7);
    }
    if (!waited) {
      pdl_wait();  // scratch is free (the previous chunk's final pass completed)
      pdl_release();
      tl_mark(tl, 1);
      waited = true;
    }
    HCLK(8);
    const int64_t rr = u / NC;
    const int c = (int)(u % NC);
    const int b = c | (LP == 1 ? (bl << 3) : (((bl & 1) << 3) | ((bl >> 1) << 2)));
    Cx<T>* dst = scratch + ((int64_t)rr << S) + ((int64_t)b << SQ) + tt;
    if (bulk) {
      // the last pass stored position pi (cf_spos = the inverse of perm): each b
      // value's block leaves as one bulk copy, read by the async proxy while
      // the transform threads start the next unit
      if (tid == issuer) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
          if (SFFT_HEAD_GROUPS && j != bl) continue;
          const int bj = c | (LP == 1 ? (j << 3) : (((j & 1) << 3) | ((j >> 1) << 2)));
#if SFFT_SCR_HINT
          // scratch is read once more, by this chunk's final pass: keep it in L2
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                       :: "l"(scratch + ((int64_t)rr << S) + ((int64_t)bj << SQ)), "r"(smem_addr(work + j * NQ)),
                          "n"(NQ * (int)sizeof(Cx<T>)), "l"(l2_policy_evict_last()) : "memory");
#else
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       :: "l"(scratch + ((int64_t)rr << S) + ((int64_t)bj << SQ)), "r"(smem_addr(work + j * NQ)),
                          "n"(NQ * (int)sizeof(Cx<T>)) : "memory");
#endif
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (cf_ppos) {
#pragma unroll
      for (int n = 0; n < E; ++n) dst[n * TPB] = sb[__ldg(cf_ppos + tt + n * TPB)];
    } else {
#pragma unroll
      for (int n = 0; n < E; ++n) dst[n * TPB] = sb[swz<T, SQ>(__ldg(perm + tt + n * TPB))];
    }
    HCLK(9);
  }
  if (bulk && tid == issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef SFFT_HEAD_CLK
  if (blockIdx.x == 0 && (tid == 0 || tid == NT - 32))
    printf("[head clk] warp %d units %u: wait_full %lld land_rd+sync %lld p0math %lld p0sts %lld sync %lld "
           "p12 lds+math %lld sts %lld sync %lld pdl %lld epi %lld loop %lld\n", tid >> 5, it, hacc[0] / it, hacc[1] / it,
           hacc[2] / it, hacc[3] / it, hacc[4] / it, hacc[5] / it, hacc[6] / it, hacc[7] / it, hacc[8] / it, hacc[9] / it,
           hacc[11] / it);
#endif
  tl_mark(tl, 2);
}

// In-place variant (SFFT_HEAD_IP=1): the landing buffer is also the working
// buffer (64 KB + 32 KB of twiddles), so two CTAs share an SM and overlap
// each other's phases; the next unit's copies are issued (by lane 0 of every
// warp, NW-th share each) once the epilogue has read the buffer.
template <typename T, int S, int P>
struct HeadIpGeo {
  using HG = HeadGeo<T, S, P>;
  static constexpr size_t SMEM = (size_t)P * HG::NQ * sizeof(Cx<T>) + (size_t)HG::NTW * sizeof(Cx<T>) + 16;
};

template <typename T, int S, int P>
__global__ void __launch_bounds__(HeadGeo<T, S, P>::NT, 2)
k_head_ip(const __grid_constant__ CUtensorMap tm, const HeadTma ht, const FrontTw2 ftw, const Cx<T>* __restrict__ tw,
          const int32_t* __restrict__ perm, Cx<T>* __restrict__ scratch, int64_t row0, int64_t units) {
  using HG = HeadGeo<T, S, P>;
  constexpr int SQ = HG::SQ, NQ = HG::NQ, E = HG::E, LE = HG::LE, TPB = HG::TPB, NT = HG::NT, NC = HG::NC;
  constexpr int LP = P == 4 ? 2 : 1, NW = NT / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Cx<T>* land = reinterpret_cast<Cx<T>*>(smem_raw);  // P x NQ: TMA box order, then swizzled slots per b value
  Cx<T>* stw = land + P * NQ;                        // twiddles of stages 5 .. SQ
  const uint32_t full = smem_addr(stw + HG::NTW);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(full, NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t u) {  // lane 0 of warp w: copies o = w, w + NW, ... of unit u
    const int w = tid >> 5;
    const int box = (NQ / ht.nops) * P;
    const int mine = ht.nops > w ? (ht.nops - w + NW - 1) / NW : 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(full), "r"((uint32_t)(mine * box * sizeof(Cx<T>))) : "memory");
    const int64_t rr = u / NC;
    const int c = (int)(u % NC);
    uint32_t offc = 0;
#pragma unroll
    for (int j = 0; j < 4 - LP; ++j)
      if ((c >> j) & 1) offc += ht.dfix[j];
    for (int o = w; o < ht.nops; o += NW) {
      uint32_t e = offc;
      for (int j = 0; j < ht.nleft; ++j)
        if ((o >> j) & 1) e += ht.left_d[j];
      const int c0 = (int)(e & ((1u << ht.k1) - 1u));
      const int c1 = (int)((e >> ht.k1) & ((1u << (ht.k2 - ht.k1)) - 1u));
      const int c2 = (int)((e >> ht.k2) & ((1u << (ht.k3 - ht.k2)) - 1u));
      const int c3 = (int)(e >> ht.k3);
      const int c4 = (int)(row0 + rr);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          :: "r"(smem_addr(land + (size_t)o * box)), "l"(&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
             "r"(full) : "memory");
    }
  };
  if ((tid & 31) == 0 && blockIdx.x < units) issue(blockIdx.x);  // signals are read-only
  for (int i = tid; i < HG::NTW; i += NT) cp_async_elem(stw + i, tw + 15 + i);
  cp_async_commit();
  const int bl = (tid >> 4) & (P - 1), tt = (tid & 15) | ((tid >> (4 + LP)) << 4);
  uint32_t qt = 0, base = 0;
#pragma unroll
  for (int i = 0; i < SQ - LE; ++i)
    if ((tt >> i) & 1) {
      qt |= 1u << ht.tq[i];
      base += ht.qw[ht.tq[i]];
    }
  const int tb0 = swz<T, SQ>((int)qt);
  Cx<T>* sb = land + bl * NQ;
  cp_async_wait<0>();
  bool waited = false;
  uint32_t it = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++it) {
    Cx<T> v[E];
    mbar_wait(full, it & 1);
#pragma unroll
    for (int x = 0; x < E; ++x) {
      uint32_t q = base;
#pragma unroll
      for (int i = 0; i < LE; ++i)
        if ((x >> i) & 1) q += ht.qw[i];
      v[x] = land[q * P + bl];
    }
    __syncthreads();  // landing reads done (and, the first time, the tables staged)
#pragma unroll
    for (int beta = 0; beta < LE; ++beta) {
#pragma unroll
      for (int x = 0; x < E; ++x) {
        if (x & (1 << beta)) continue;
        const int j = (1 << beta) - 1 + (x & ((1 << beta) - 1));
        bfly2(v[x], v[x | (1 << beta)], ftw.w[j], ftw.iw[j]);
      }
    }
#pragma unroll
    for (int x = 0; x < E; ++x) sb[tb0 ^ swz<T, SQ>(x)] = v[x];
    __syncthreads();
#pragma unroll
    for (int p = 1; p < HG::NPASS; ++p) {
      const int tb = swz<T, SQ>(slot_t<SQ, LE>(p, tt));
#pragma unroll
      for (int x = 0; x < E; ++x) v[x] = sb[tb ^ swz<T, SQ>(slot_x<SQ, LE>(p, x))];
      const int b0 = p * LE, b1 = (b0 + LE < SQ) ? b0 + LE : SQ, w0 = pass_w0(p, SQ, LE);
#pragma unroll
      for (int beta = b0; beta < b1; ++beta) {
        const int lb = beta - w0;
#pragma unroll
        for (int xl = 0; xl < (1 << lb); ++xl) {
          const int a0 = slot_of<SQ, LE>(p, tt, xl);
          const Cx<T> w = stw[(1 << beta) - 16 + (a0 & ((1 << beta) - 1))];
          const Cx<T> iw = rot_i(w);
#pragma unroll
          for (int x = xl; x < E; x += (1 << lb)) {
            if (x & (1 << lb)) continue;
            bfly2(v[x], v[x | (1 << lb)], w, iw);
          }
        }
      }
#pragma unroll
      for (int x = 0; x < E; ++x) sb[tb ^ swz<T, SQ>(slot_x<SQ, LE>(p, x))] = v[x];
      __syncthreads();
    }
#pragma unroll
    for (int n = 0; n < E; ++n) v[n] = sb[swz<T, SQ>(__ldg(perm + tt + n * TPB))];
    __syncthreads();  // the buffer is free: the next unit's copies may land
    if ((tid & 31) == 0 && u + gridDim.x < units) issue(u + gridDim.x);
    if (!waited) {
      pdl_wait();  // scratch is free (the previous chunk's final pass completed)
      pdl_release();
      waited = true;
    }
    const int64_t rr = u / NC;
    const int c = (int)(u % NC);
    const int b = c | (LP == 1 ? (bl << 3) : (((bl & 1) << 3) | ((bl >> 1) << 2)));
    Cx<T>* dst = scratch + ((int64_t)rr << S) + ((int64_t)b << SQ) + tt;
#pragma unroll
    for (int n = 0; n < E; ++n) dst[n * TPB] = v[n];
  }
}

// Final pass of the head path: as k_tri_final (a thread owns position pi for
// the rows of its CTA; 15 twiddles per pi, last 4 stages in registers) with
// FFMA2 butterflies and, when the plan's output map is blocked (output of
// slot (b, q) at T * 2^(S-4) + pi(q) for a per-q bijection b -> T: config 5,
// whose top four pivots are the top bits of j), stores staged per warp in
// shared memory so that each store instruction writes 32 consecutive
// outputs of one block T instead of 32 scattered ones.
template <typename T, int S>
struct Fin2Geo {
  static constexpr int L = 4, EXL = 16, SQ = S - L, NQ = 1 << SQ, NT = 128, NW = NT / 32, NQB = NQ / NT;
  static constexpr size_t SMEM = 2 * (size_t)NW * EXL * 32 * sizeof(Cx<T>);  // output staging, two buffers per warp
};

#ifndef SFFT_FIN2_MINB  // resident final-pass CTAs per SM the register budget is set for
#define SFFT_FIN2_MINB 4
#endif
#ifndef SFFT_FIN2_NOPF
#define SFFT_FIN2_NOPF 0
#endif
template <typename T, int S>
__global__ void __launch_bounds__(128, SFFT_FIN2_MINB) k_fin2(const PlanArgs args, const Cx<T>* __restrict__ scr2, int64_t row0,
                                                 int64_t nrows, int nper, const Cx<T>* __restrict__ twf,
                                                 const int32_t* __restrict__ invf, const int32_t* __restrict__ perm,
                                                 int blocked, const __grid_constant__ CUtensorMap otm, int tmaout,
                                                 unsigned long long* tl) {
  tl_mark(tl, 0);
  using FG = Fin2Geo<T, S>;
  constexpr int NQ = FG::NQ, SQ = FG::SQ, EXL = FG::EXL, L = FG::L, NT = FG::NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Cx<T>* stg = reinterpret_cast<Cx<T>*>(smem_raw);  // [warp][buffer][T][lane] output staging
  const int qb = blockIdx.x % FG::NQB;
  const int64_t first = blockIdx.x / FG::NQB;
  if (first >= nrows) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pi = qb * NT + threadIdx.x;
  Cx<T>* st = stg + wid * 2 * EXL * 32;
  uint32_t sbuf = 0;
  Cx<T> nx[EXL];
  auto fetch = [&](int64_t rr) {
    const Cx<T>* src = scr2 + (rr << S) + pi;
#pragma unroll
    for (int b = 0; b < EXL; ++b) nx[b] = ld_cs(src + ((int64_t)b << SQ));
  };
  const int q = perm[pi];
  // this thread's 15 twiddles in registers, i*w formed per use, and (blocked)
  // the block T of value b in 4-bit fields (config 5 per step: twiddles and
  // i*twiddles in shared memory 124.7 us, twiddles only 121.8, registers 120.7)
  Cx<T> wr[EXL - 1];
#pragma unroll
  for (int j = 0; j < EXL - 1; ++j) wr[j] = twf[(int64_t)j * NQ + pi];
  uint64_t epk = 0;
  if (blocked) {
#pragma unroll
    for (int b = 0; b < EXL; ++b)
      epk |= (uint64_t)((invf ? invf[(int64_t)b * NQ + pi] : ((b << SQ) | q)) >> SQ) << (4 * b);
  }
  pdl_wait();  // scratch written by this chunk's head pass
  pdl_release();
  tl_mark(tl, 1);
  fetch(first);
  const T scale = (T)args.scale1;
  const int pib = qb * NT + wid * 32;  // this warp's first pi
#ifdef SFFT_HEAD_CLK
  long long hacc[12] = {0}, hlast = clock64();
  int it = 0;
#endif
  for (int64_t rr = first; rr < nrows; rr += nper) {
    Cx<T> v[EXL];
#ifdef SFFT_HEAD_CLK
    ++it;
    {
      float acc = 0.f;
#pragma unroll
      for (int b = 0; b < EXL; ++b) acc += nx[b].x;
      if (acc == 12345.678f) printf("x");
    }
    HCLK(0);
#endif
#if SFFT_FIN2_NOPF  // no register prefetch of the next row: fewer registers, more resident CTAs
    if (rr != first) fetch(rr);
#pragma unroll
    for (int b = 0; b < EXL; ++b) v[b] = nx[b];
#else
#pragma unroll
    for (int b = 0; b < EXL; ++b) v[b] = nx[b];
#if defined(SFFT_FIN_PROBE) && SFFT_FIN_PROBE == 1  // timing probe: no scratch loads after the first row
    if (false)
#endif
    if (rr + nper < nrows) fetch(rr + nper);
#endif
    HCLK(1);
#pragma unroll
    for (int t = 0; t < L; ++t) {  // global stage SQ + t + 1 pairs slot bit SQ + t = b bit t
#pragma unroll
      for (int b = 0; b < EXL; ++b) {
        if (b & (1 << t)) continue;
        const int j = (1 << t) - 1 + (b & ((1 << t) - 1));
        const Cx<T> w = wr[j];
        bfly2(v[b], v[b | (1 << t)], w, rot_i(w));
      }
    }
    const int64_t r = row0 + rr;
    Cx<T>* o1 = reinterpret_cast<Cx<T>*>(args.out1) + r * args.ld1;
    HCLK(2);
#if defined(SFFT_FIN_PROBE) && SFFT_FIN_PROBE == 2  // timing probe: no output stores
    if (v[0].x == 12345.678f)
#endif
    if (blocked && tmaout) {
      // the warp's 16 x 32 outputs leave as one tensor store (box: 32 pi x 16
      // blocks T of row r), read by the async proxy while the warp works on
      // the next row in the other staging buffer
      Cx<T>* sw = st + sbuf * EXL * 32;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // buffer sbuf's previous store was read
      __syncwarp();
#pragma unroll
      for (int b = 0; b < EXL; ++b) sw[(int)((epk >> (4 * b)) & 15) * 32 + lane] = cscale(v[b], scale);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
#if SFFT_OUT_HINT
        // outputs are not read again by this call: first out of L2
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
                     :: "l"(&otm), "r"(pib), "r"(0), "r"((int)r), "r"(smem_addr(sw)), "l"(l2_policy_evict_first())
                     : "memory");
#else
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                     :: "l"(&otm), "r"(pib), "r"(0), "r"((int)r), "r"(smem_addr(sw)) : "memory");
#endif
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      sbuf ^= 1;
    } else if (blocked) {
#pragma unroll
      for (int b = 0; b < EXL; ++b) st[(int)((epk >> (4 * b)) & 15) * 32 + lane] = cscale(v[b], scale);
      __syncwarp();
      HCLK(3);
#pragma unroll
      for (int t = 0; t < EXL; ++t) st_cs(o1 + ((int64_t)t << SQ) + pib + lane, st[t * 32 + lane]);
      __syncwarp();
      HCLK(4);
    } else {
#pragma unroll
      for (int b = 0; b < EXL; ++b) {
        const int eb = invf ? __ldg(invf + (int64_t)b * NQ + pi) : ((b << SQ) | q);
        st_cs_if(o1, eb, cscale(v[b], scale));
      }
    }
    if (args.out2) {
      Cx<T>* o2 = reinterpret_cast<Cx<T>*>(args.out2) + r * args.ld2;
#pragma unroll
      for (int b = 0; b < EXL; ++b) o2[(b << SQ) | q] = v[b];
    }
  }
  if (tmaout && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#ifdef SFFT_HEAD_CLK
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
    printf("[fin clk] warp %d iters %d: wait_nx %lld issue_fetch %lld math %lld stage %lld store %lld\n", wid, it,
           hacc[0] / it, hacc[1] / it, hacc[2] / it, hacc[3] / it, hacc[4] / it);
#endif
  tl_mark(tl, 2);
}

// Final pass with both directions asynchronous (blocked output maps only):
// a warp's 32 pi x 16 b values of a row arrive by one tensor load (box 32 x
// 16 x 1 of the scratch viewed as [pi, b, row]) into a two-slot ring, two
// rows ahead of the butterflies, and leave by one tensor store as in k_fin2;
// the thread keeps only its 16 values and 15 twiddles in registers.
#ifndef SFFT_FIN3_MINB
#define SFFT_FIN3_MINB 4
#endif
template <typename T, int S>
struct Fin3Geo {
  static constexpr int L = 4, EXL = 16, SQ = S - L, NQ = 1 << SQ, NT = 128, NW = NT / 32, NQB = NQ / NT;
  static constexpr int TILE = EXL * 32;  // values per warp and row
  // per warp: 2 landing slots + 1 output staging tile; then 2 mbarriers per warp
  static constexpr size_t SMEM = (size_t)NW * 3 * TILE * sizeof(Cx<T>) + (size_t)NW * 2 * 8;
};

template <typename T, int S>
__global__ void __launch_bounds__(128, SFFT_FIN3_MINB)
k_fin3(const PlanArgs args, const __grid_constant__ CUtensorMap itm, const __grid_constant__ CUtensorMap otm,
       int64_t row0, int64_t nrows, int nper, const Cx<T>* __restrict__ twf, const int32_t* __restrict__ invf,
       const int32_t* __restrict__ perm, unsigned long long* tl) {
  tl_mark(tl, 0);
  using FG = Fin3Geo<T, S>;
  constexpr int NQ = FG::NQ, SQ = FG::SQ, EXL = FG::EXL, L = FG::L, NT = FG::NT, TILE = FG::TILE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int qb = blockIdx.x % FG::NQB;
  const int64_t first = blockIdx.x / FG::NQB;
  if (first >= nrows) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int pi = qb * NT + threadIdx.x;
  const int pib = qb * NT + wid * 32;  // this warp's first pi
  Cx<T>* in = reinterpret_cast<Cx<T>*>(smem_raw) + (size_t)wid * 3 * TILE;  // [slot][b][lane]
  Cx<T>* ob = in + 2 * TILE;                                                 // [T][lane]
  const uint32_t bar0 = smem_addr(reinterpret_cast<Cx<T>*>(smem_raw) + (size_t)FG::NW * 3 * TILE) + 16 * wid;
  if (lane == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int q = perm[pi];
  Cx<T> wr[EXL - 1];
#pragma unroll
  for (int j = 0; j < EXL - 1; ++j) wr[j] = twf[(int64_t)j * NQ + pi];
  uint64_t epk = 0;
#pragma unroll
  for (int b = 0; b < EXL; ++b)
    epk |= (uint64_t)((invf ? invf[(int64_t)b * NQ + pi] : ((b << SQ) | q)) >> SQ) << (4 * b);
  pdl_wait();  // scratch written by this chunk's head pass
  pdl_release();
  tl_mark(tl, 1);
  auto load = [&](int64_t rr, int slot) {  // lane 0: the warp's tile of scratch row rr into ring slot `slot`
    const uint32_t bar = bar0 + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(bar), "r"((uint32_t)(TILE * sizeof(Cx<T>))) : "memory");
#if SFFT_FIN_LOAD_HINT
    // probe: scratch rows are dead once read
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
        :: "r"(smem_addr(in + slot * TILE)), "l"(&itm), "r"(pib), "r"(0), "r"((int)rr), "r"(bar),
           "l"(l2_policy_evict_first()) : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(smem_addr(in + slot * TILE)), "l"(&itm), "r"(pib), "r"(0), "r"((int)rr), "r"(bar) : "memory");
#endif
  };
  if (lane == 0) {
    load(first, 0);
    if (first + nper < nrows) load(first + nper, 1);
  }
  const T scale = (T)args.scale1;
  uint32_t it = 0;
  for (int64_t rr = first; rr < nrows; rr += nper, ++it) {
    const int slot = it & 1;
    mbar_wait(bar0 + 8 * slot, (it >> 1) & 1);
    Cx<T> v[EXL];
#pragma unroll
    for (int b = 0; b < EXL; ++b) v[b] = in[slot * TILE + b * 32 + lane];
#pragma unroll
    for (int t = 0; t < L; ++t) {  // global stage SQ + t + 1 pairs slot bit SQ + t = b bit t
#pragma unroll
      for (int b = 0; b < EXL; ++b) {
        if (b & (1 << t)) continue;
        const int j = (1 << t) - 1 + (b & ((1 << t) - 1));
        const Cx<T> w = wr[j];
        bfly2(v[b], v[b | (1 << t)], w, rot_i(w));
      }
    }
    // the slot's values are in registers (consumed above): refill it two rows ahead
    __syncwarp();
    if (lane == 0) {
      if (rr + 2 * (int64_t)nper < nrows) load(rr + 2 * (int64_t)nper, slot);
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the previous row's store has read `ob`
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < EXL; ++b) ob[(int)((epk >> (4 * b)) & 15) * 32 + lane] = cscale(v[b], scale);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
#if SFFT_OUT_HINT
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
                   :: "l"(&otm), "r"(pib), "r"(0), "r"((int)(row0 + rr)), "r"(smem_addr(ob)),
                      "l"(l2_policy_evict_first()) : "memory");
#else
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                   :: "l"(&otm), "r"(pib), "r"(0), "r"((int)(row0 + rr)), "r"(smem_addr(ob)) : "memory");
#endif
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tl_mark(tl, 2);
}

// host: the tensor-map decomposition of a plan's pattern (false: not eligible)
static bool head_plan(const sfft_plan* p, int P, HeadTma* ht) {
  const int S = p->s, M = p->M, SQ = S - 4;
  if (S < 12 || S > 20) return false;
  std::memset(ht, 0, sizeof(*ht));
  ht->P = P;
  auto d = [&](int i) { return M - 1 - p->used[i]; };  // log2 of slot bit i's sample stride
  if (d(S - 1) != 0 || (P == 4 && d(S - 2) != 1)) return false;
  const int LP = P == 4 ? 2 : 1;
  for (int j = 0; j < 4 - LP; ++j) ht->dfix[j] = 1u << d(SQ + j);
  // runs of q bits with consecutive strides: q bit i has log-stride d(i), decreasing in i
  struct Run { int lo, len; };  // element-offset bits [lo, lo+len)
  std::vector<Run> runs;
  for (int i = SQ - 1; i >= 0;) {
    int j = i;
    while (j - 1 >= 0 && d(j - 1) == d(j) + 1 && (i - j + 1) < 8) --j;
    runs.push_back({d(i), i - j + 1});
    i = j - 1;
  }
  std::vector<int> idx(runs.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return runs[a].len > runs[b].len; });
  std::vector<Run> pick;
  for (size_t i = 0; i < idx.size() && pick.size() < 3; ++i) pick.push_back(runs[idx[i]]);
  std::sort(pick.begin(), pick.end(), [](const Run& a, const Run& b) { return a.lo < b.lo; });
  while (pick.size() < 3) pick.push_back({M, 0});
  ht->k1 = pick[0].lo;
  ht->k2 = pick[1].lo;
  ht->k3 = pick[2].lo;
  if (ht->k1 < (uint32_t)LP) return false;
  int boxq = 0;
  for (int j = 0; j < 3; ++j) {
    ht->len[j] = pick[j].len;
    boxq += pick[j].len;
  }
  if (boxq < 3) return false;  // landing boxes of >= 128 B
  // landing weights: run bits in box order, then the enumerated bits
  int wpos = 0;
  for (int j = 0; j < 3; ++j)
    for (int t = 0; t < pick[j].len; ++t) {
      const int e = pick[j].lo + t;
      for (int i = 0; i < SQ; ++i)
        if (d(i) == e) ht->qw[i] = 1u << (wpos + t);
    }
  for (int j = 0, w = 0; j < 3; ++j) {  // box order: run 0 lowest
    for (int t = 0; t < pick[j].len; ++t)
      for (int i = 0; i < SQ; ++i)
        if (d(i) == pick[j].lo + t) ht->qw[i] = 1u << (w + t);
    w += pick[j].len;
  }
  wpos = boxq;
  for (int i = 0; i < SQ; ++i) {
    bool in_run = false;
    for (int j = 0; j < 3; ++j) in_run |= d(i) >= pick[j].lo && d(i) < pick[j].lo + pick[j].len;
    if (in_run) continue;
    ht->left_d[ht->nleft] = 1u << d(i);
    ht->qw[i] = 1u << (wpos + ht->nleft);
    ++ht->nleft;
  }
  ht->nops = 1 << ht->nleft;
  std::vector<int> qb;
  for (int i = 4; i < SQ; ++i) qb.push_back(i);
  std::stable_sort(qb.begin(), qb.end(), [&](int a, int b) { return ht->qw[a] < ht->qw[b]; });
  for (size_t i = 0; i < qb.size(); ++i) ht->tq[i] = (uint8_t)qb[i];
  return ht->nleft <= 10;
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

template <typename T, int S, int P>
static int head_launches(int64_t rows, int64_t* n) {
  const int64_t chunk = tri_chunk_rows(rows, sizeof(Cx<T>) << S);
  *n = rows > 0 ? 2 * ((rows + chunk - 1) / chunk) : 0;
  return SFFT_OK;
}

// SFFT_TIMELINE: launch records (start, past wait, end) printed at exit
struct Timeline {
  unsigned long long* d = nullptr;
  std::vector<std::string> names;
  static constexpr int kSlots = 4096;
  ~Timeline() {
    if (!d || names.empty()) return;
    std::vector<unsigned long long> h(3 * (size_t)kSlots);
    if (cudaMemcpy(h.data(), d, 8 * h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    const unsigned long long t0 = h[0];
    for (size_t i = 0; i < names.size() && i < (size_t)kSlots; ++i)
      fprintf(stderr, "[sfft timeline] %4zu %-6s start %10.2f us  past-wait %10.2f us  end %10.2f us\n", i,
              names[i].c_str(), (h[3 * i] - t0) * 1e-3, (h[3 * i + 1] - t0) * 1e-3, (h[3 * i + 2] - t0) * 1e-3);
  }
};
static Timeline g_tl;
static std::mutex g_tl_mu;
static unsigned long long* timeline_slot(const char* name) {
  static const bool on = getenv("SFFT_TIMELINE") != nullptr;
  if (!on) return nullptr;
  std::lock_guard<std::mutex> lk(g_tl_mu);
  if (!g_tl.d) {
    if (cudaMalloc(&g_tl.d, 8 * 3 * (size_t)Timeline::kSlots) != cudaSuccess) return nullptr;
    std::vector<unsigned long long> init(3 * (size_t)Timeline::kSlots);
    for (size_t i = 0; i < init.size(); ++i) init[i] = (i % 3 == 2) ? 0ull : ~0ull;
    cudaMemcpy(g_tl.d, init.data(), 8 * init.size(), cudaMemcpyHostToDevice);
  }
  if (g_tl.names.size() >= (size_t)Timeline::kSlots) return nullptr;
  g_tl.names.push_back(name);
  return g_tl.d + 3 * (g_tl.names.size() - 1);
}

// 1: launched; 0: not eligible (caller falls back); <0 never; >1 error code
template <typename T, int S, int P>
static int run_head(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st, bool* ran) {
  using HG = HeadGeo<T, S, P>;
  *ran = false;
  HeadTma ht;
  if (!p->d_tri_perm || a.identity != 0 || a.nshift != 1 || a.negshift != 0 || a.in_c64 || a.debug_skip ||
      (reinterpret_cast<uintptr_t>(a.sig) & 15) || ((a.ld * (int64_t)sizeof(Cx<T>)) & 15) || a.B > 0x7fffffff ||
      !head_plan(p, P, &ht))
    return SFFT_OK;
  const int32_t* invf = inv1 == p->d_inv_elem ? p->d_tri_inv_elem
                        : inv1 == p->d_inv_node ? p->d_tri_inv_node
                                                : nullptr;
  if (inv1 && !invf) return SFFT_OK;
  auto enc = tensor_map_encoder();
  if (!enc) return SFFT_OK;
  CUtensorMap tm;
  const cuuint64_t dims[5] = {(cuuint64_t)1 << ht.k1, (cuuint64_t)1 << (ht.k2 - ht.k1),
                              (cuuint64_t)1 << (ht.k3 - ht.k2), (cuuint64_t)1 << (a.M - ht.k3), (cuuint64_t)a.B};
  const cuuint64_t strides[4] = {(cuuint64_t)sizeof(Cx<T>) << ht.k1, (cuuint64_t)sizeof(Cx<T>) << ht.k2,
                                 (cuuint64_t)sizeof(Cx<T>) << ht.k3, (cuuint64_t)(a.ld * (int64_t)sizeof(Cx<T>))};
  const cuuint32_t box[5] = {(cuuint32_t)P, 1u << ht.len[0], 1u << ht.len[1], 1u << ht.len[2], 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 5, const_cast<void*>(a.sig), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SFFT_OK;
  auto head = k_head<T, S, P>;
  auto fin = k_fin2<T, S>;
  using FG = Fin2Geo<T, S>;
  int occ1 = 0, occ3 = 0, rc;
  // a variant that does not fit on an SM (e.g. SFFT_HEAD_P=4: 288 KB of
  // shared memory) leaves the call to the three-pass split
  auto soft = [](int r) { return r == SFFT_ERR_UNSUPPORTED ? -1 : r; };
  if ((rc = soft(kernel_occupancy(head, HG::NTT, HG::SMEM, &occ1)))) return rc < 0 ? SFFT_OK : rc;
  static const bool ip = [] {
    const char* e = getenv("SFFT_HEAD_IP");
    return e && atoi(e) == 1;
  }();
  // SFFT_HEAD_BULK=0: the epilogue reads the working buffer through perm and
  // stores from registers; default: bulk copies (cp.async.bulk shared -> global)
  static const bool bulk = [] {
    const char* e = getenv("SFFT_HEAD_BULK");
    return !(e && atoi(e) == 0);
  }();
  auto head_ip = k_head_ip<T, S, P>;
  int occ_ip = 0;
  if (ip && (rc = soft(kernel_occupancy(head_ip, HG::NT, HeadIpGeo<T, S, P>::SMEM, &occ_ip))))
    return rc < 0 ? SFFT_OK : rc;
  if ((rc = soft(kernel_occupancy(fin, FG::NT, FG::SMEM, &occ3)))) return rc < 0 ? SFFT_OK : rc;
  const int blocked = inv1 == p->d_inv_elem ? p->tri_blocked_elem : inv1 == p->d_inv_node ? p->tri_blocked_node : 0;
  // blocked output map: each final-pass warp writes its 32 pi x 16 blocks of a
  // row with one tensor store (SFFT_FIN_TMA=0: staged per-thread stores)
  static const bool fin_tma = [] {
    const char* e = getenv("SFFT_FIN_TMA");
    return !(e && atoi(e) == 0);
  }();
  CUtensorMap otm;
  std::memset(&otm, 0, sizeof(otm));
  int tmaout = 0;
  if (blocked && fin_tma && !a.out2 && a.n1 == ((int64_t)1 << S) && !(reinterpret_cast<uintptr_t>(a.out1) & 15) &&
      !((a.ld1 * (int64_t)sizeof(Cx<T>)) & 15)) {
    const cuuint64_t od[3] = {(cuuint64_t)HG::NQ, 16, (cuuint64_t)a.B};
    const cuuint64_t os[2] = {(cuuint64_t)sizeof(Cx<T>) << HG::SQ, (cuuint64_t)(a.ld1 * (int64_t)sizeof(Cx<T>))};
    const cuuint32_t ob[3] = {32, 16, 1};
    const cuuint32_t oe[3] = {1, 1, 1};
    tmaout = enc(&otm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, a.out1, od, os, ob, oe, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  *ran = true;
  const int64_t rows = a.B;
  if (rows == 0) return SFFT_OK;
  const size_t row_bytes = sizeof(Cx<T>) << S;
  const int64_t chunk = tri_chunk_rows(rows, row_bytes);
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  void* scr = nullptr;
  bool pooled = false;
  if ((rc = stream_scratch(dev, st, (size_t)chunk * row_bytes, &scr, &pooled))) return rc;
  const Cx<T>* tw = reinterpret_cast<const Cx<T>*>(p->d_twiddles);
  const Cx<T>* twf = reinterpret_cast<const Cx<T>*>(p->d_tri_tw);
  const int64_t sms = num_sms();
  FrontTw2 ftw;
  std::memcpy(ftw.w, p->tri_front_tw, sizeof(Cx<float>) * 15);
  for (int j = 0; j < 15; ++j) ftw.iw[j] = Cx<float>{-ftw.w[j].y, ftw.w[j].x};
  static const bool pdl = [] {
    const char* e = getenv("SFFT_TRI_PDL");
    return !(e && atoi(e) == 0);
  }();
  const ByteRange in[1] = {{(uintptr_t)a.sig, (uintptr_t)a.sig + (size_t)((a.B - 1) * a.ld + (1ll << a.M)) * sizeof(Cx<T>)}};
  const ByteRange outs[2] = {
      {(uintptr_t)a.out1, (uintptr_t)a.out1 + (size_t)((rows - 1) * a.ld1 + a.n1) * sizeof(Cx<T>)},
      {(uintptr_t)a.out2, a.out2 ? (uintptr_t)a.out2 + (size_t)((rows - 1) * a.ld2 + (1ll << S)) * sizeof(Cx<T>) : 0}};
  const bool pdl_first = pdl_join(st, in, 1, outs, 2, pdl && !pooled);
  // final pass with tensor loads as well (k_fin3, under the tensor-store conditions; SFFT_FIN3=0: k_fin2)
  static const bool fin3_on = [] {
    const char* e = getenv("SFFT_FIN3");
    return !(e && atoi(e) == 0);
  }();
  using F3 = Fin3Geo<T, S>;
  auto fin3 = k_fin3<T, S>;
  int occ_f3 = 0;
  CUtensorMap itm;
  std::memset(&itm, 0, sizeof(itm));
  bool use_fin3 = false;
  if (fin3_on && tmaout && soft(kernel_occupancy(fin3, F3::NT, F3::SMEM, &occ_f3)) == 0 && occ_f3 > 0) {
    const cuuint64_t id[3] = {(cuuint64_t)HG::NQ, 16, (cuuint64_t)chunk};
    const cuuint64_t is[2] = {(cuuint64_t)sizeof(Cx<T>) << HG::SQ, (cuuint64_t)sizeof(Cx<T>) << S};
    const cuuint32_t ib[3] = {32, 16, 1};
    const cuuint32_t ie[3] = {1, 1, 1};
    use_fin3 = enc(&itm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, scr, id, is, ib, ie, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cudaError_t e = cudaSuccess;
  for (int64_t r0 = 0; r0 < rows && e == cudaSuccess; r0 += chunk) {
    const int64_t n = std::min(chunk, rows - r0);
    const int64_t units = n * HG::NC;
    if (ip)
      e = launch_k(head_ip, (unsigned)std::min<int64_t>(units, sms * occ_ip), HG::NT, HeadIpGeo<T, S, P>::SMEM, st,
                   pdl && (r0 > 0 || pdl_first), tm, ht, ftw, tw, (const int32_t*)p->d_tri_perm, (Cx<T>*)scr, r0,
                   units);
    else
      e = launch_k(head, (unsigned)std::min<int64_t>(units, sms * occ1), HG::NTT, HG::SMEM, st,
                   pdl && (r0 > 0 || pdl_first), tm, ht, ftw, tw, (const int32_t*)p->d_tri_perm, (Cx<T>*)scr, r0,
                   units, (const int32_t*)(bulk ? p->d_tri_pinv : P == 2 ? p->d_head_spos : nullptr),
                   (const int32_t*)(bulk ? nullptr : P == 2 ? p->d_head_ppos : nullptr), (int)bulk,
                   timeline_slot("head"));
    int nper = (int)std::max<int64_t>(1, std::min<int64_t>(n, sms * occ3 / FG::NQB));
    static const int nper_env = [] {
      const char* e = getenv("SFFT_FIN_NPER");
      return e ? atoi(e) : 0;
    }();
    if (nper_env > 0) nper = (int)std::min<int64_t>(n, nper_env);  // probe: more, shorter final-pass CTAs
    if (e == cudaSuccess && use_fin3) {
      const int nper3 = (int)std::max<int64_t>(1, std::min<int64_t>(n, sms * occ_f3 / F3::NQB));
      e = launch_k(fin3, (unsigned)(nper3 * F3::NQB), F3::NT, F3::SMEM, st, pdl, a, itm, otm, r0, n, nper3, twf,
                   invf, (const int32_t*)p->d_tri_perm, timeline_slot("fin"));
    } else if (e == cudaSuccess)
      e = launch_k(fin, (unsigned)(nper * FG::NQB), FG::NT, FG::SMEM, st, pdl, a, (const Cx<T>*)scr, r0, n, nper, twf,
                   invf, (const int32_t*)p->d_tri_perm, blocked, otm, tmaout, timeline_slot("fin"));
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (pooled) cudaFreeAsync(scr, st);
  if (e != cudaSuccess) return cuda_fail(e, "head transform launch");
  return SFFT_OK;
}

// SFFT_HEAD=0 keeps the three-pass split; SFFT_HEAD_P selects the piece (2 or 4)
static int head_mode() {
  static const int v = [] {
    const char* e = getenv("SFFT_HEAD");
    if (e && atoi(e) == 0) return 0;
    const char* q = getenv("SFFT_HEAD_P");
    return (q && atoi(q) == 4) ? 4 : 2;
  }();
  return v;
}

bool split_two_pass() { return !use_tri(); }

// the plan's device-resident transforms take the head path (plan build skips
// the three-pass middle pass's conflict-free tables then)
bool head_covers(const sfft_plan* p) {
  HeadTma ht;
  return use_tri() && head_mode() == 2 && p->dtype == SFFT_C64 && p->s == 16 && head_plan(p, 2, &ht);
}

static int try_head(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st, bool* ran) {
  *ran = false;
  const int P = head_mode();
  if (P == 0 || p->dtype != SFFT_C64) return SFFT_OK;
  switch (p->s) {
    case 16: return P == 4 ? run_head<float, 16, 4>(p, a, inv1, st, ran) : run_head<float, 16, 2>(p, a, inv1, st, ran);
    default: return SFFT_OK;
  }
}


int run_large(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
  if (use_tri()) {
    bool ran = false;
    const int rc = try_head(p, a, inv1, st, &ran);
    if (rc || ran) return rc;
    if (p->dtype == SFFT_C64) {
      switch (p->s) {
        case 15: return run_tri<float, 15, 3>(p, a, inv1, st);
        case 16: return run_tri<float, 16, 4>(p, a, inv1, st);
        case 17: return run_tri<float, 17, 4>(p, a, inv1, st);
        default: break;
      }
    } else {
      switch (p->s) {
        case 14: return run_tri<double, 14, 2>(p, a, inv1, st);
        case 15: return run_tri<double, 15, 3>(p, a, inv1, st);
        case 16: return run_tri<double, 16, 4>(p, a, inv1, st);
        default: break;
      }
    }
  }
  if (p->dtype == SFFT_C64) {
    switch (p->s) {
      case 15: return run_split<float, 15, 3>(p, a, inv1, st);
      case 16: return run_split<float, 16, 4>(p, a, inv1, st);
      case 17: return run_split<float, 17, 4>(p, a, inv1, st);
      default: break;
    }
  } else {
    switch (p->s) {
      case 14: return run_split<double, 14, 2>(p, a, inv1, st);
      case 15: return run_split<double, 15, 3>(p, a, inv1, st);
      case 16: return run_split<double, 16, 4>(p, a, inv1, st);
      default: break;
    }
  }
  return fail(SFFT_ERR_UNSUPPORTED, "2^s slots exceed the device transform (s=" + std::to_string(p->s) + ")");
}

int large_launch_count(const sfft_plan* p, int64_t rows, int64_t* launches) {
  if (use_tri()) {
    HeadTma ht;
    if (head_mode() == 2 && p->dtype == SFFT_C64 && p->s == 16 && p->d_tri_perm && head_plan(p, 2, &ht))
      return head_launches<float, 16, 2>(rows, launches);
    if (p->dtype == SFFT_C64) {
      switch (p->s) {
        case 15: return tri_launches<float, 15, 3>(rows, launches);
        case 16: return tri_launches<float, 16, 4>(rows, launches);
        case 17: return tri_launches<float, 17, 4>(rows, launches);
        default: break;
      }
    } else {
      switch (p->s) {
        case 14: return tri_launches<double, 14, 2>(rows, launches);
        case 15: return tri_launches<double, 15, 3>(rows, launches);
        case 16: return tri_launches<double, 16, 4>(rows, launches);
        default: break;
      }
    }
  }
  if (p->dtype == SFFT_C64) {
    switch (p->s) {
      case 15: return split_launches<float, 15, 3>(rows, launches);
      case 16: return split_launches<float, 16, 4>(rows, launches);
      case 17: return split_launches<float, 17, 4>(rows, launches);
      default: break;
    }
  } else {
    switch (p->s) {
      case 14: return split_launches<double, 14, 2>(rows, launches);
      case 15: return split_launches<double, 15, 3>(rows, launches);
      case 16: return split_launches<double, 16, 4>(rows, launches);
      default: break;
    }
  }
  *launches = rows > 0 ? 1 : 0;
  return SFFT_OK;
}

}  // namespace sfft
