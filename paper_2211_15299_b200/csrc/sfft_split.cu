// Two-pass split transform for 2^s beyond one CTA (configs 5/6, s = 14..17):
// a front pass runs the first lc stages across 2^lc sorted blocks in
// registers and writes an L2-resident scratch; a persistent back pass runs
// the remaining s - lc stages per block in shared memory and stores through
// the block-major inverse map.  See DESIGN.md "Large A".
//
// Reference: hidft.py:135-185 (hidft), hidft.py:160-167 (butterfly).

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

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

int run_large(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st) {
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
