// Device-side support analysis and ButterflyPlan construction.
//
// Reference: congruence.py:76-101 (pivots), congruence.py:235-278 (classify,
// part-homogeneity, validate_pivot_vector), sampling.py:62-71
// (pivoted_pattern), hidft.py:69-95 (_build_plan), hidft.py:168-178 (node
// ordering).  Every index table is bit-exact with the reference.
//
// pivots(J): the split levels of the congruence tree are exactly the levels
// ctz(a ^ b) of ADJACENT pairs when J is sorted by its bit-reversed keys
// (bit-reversal turns the LSB-first trie into an ordinary sorted order, and
// every branching node of a trie is witnessed by an adjacent pair).  The
// keys are distinct M-bit integers, so the sort is a bitmap rank:
// set bits, prefix-popcount the words, rank = prefix + popc(low bits).

#include <algorithm>
#include <chrono>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sfft_common.cuh"
#include "sfft_plan.h"

namespace sfft {

// ------------------------------------------------------------ errors ---
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return SFFT_ERR_CUDA;
}

bool is_device_pointer(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged ||
         (attr.type == cudaMemoryTypeHost && attr.devicePointer == p);
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// --------------------------------------------------------- bitmap rank ---
constexpr int kScanBlock = 1024;

__global__ void k_support_keys(const int64_t* __restrict__ J, int64_t k, int M,
                               uint32_t* __restrict__ keys, uint32_t* __restrict__ bitmap,
                               int* __restrict__ status) {
  const int64_t N = 1ll << M;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = J[e];
    if (j < 0 || j >= N || (e > 0 && J[e - 1] >= j)) {
      atomicMax(status, SFFT_ERR_INVALID);
      keys[e] = 0;
      continue;
    }
    const uint32_t key = __brev((uint32_t)j) >> (32 - M);
    keys[e] = key;
    atomicOr(&bitmap[key >> 5], 1u << (key & 31));
  }
}

__global__ void k_set_bits(const uint32_t* __restrict__ keys, const uint8_t* __restrict__ valid,
                           int64_t n, uint32_t* __restrict__ bitmap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (valid && !valid[i]) continue;
    const uint32_t key = keys[i];
    atomicOr(&bitmap[key >> 5], 1u << (key & 31));
  }
}

// block-exclusive prefix of popcounts over kScanBlock words
__global__ void __launch_bounds__(kScanBlock)
k_word_scan(const uint32_t* __restrict__ bitmap, int64_t nwords, uint32_t* __restrict__ wprefix,
            uint32_t* __restrict__ bsum) {
  __shared__ uint32_t warp_tot[kScanBlock / 32];
  const int64_t w = blockIdx.x * (int64_t)kScanBlock + threadIdx.x;
  const uint32_t c = w < nwords ? __popc(bitmap[w]) : 0u;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = warp_tot[lane];
    uint32_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += y;
    }
    warp_tot[lane] = xi - x;  // exclusive warp offsets
    if (lane == 31) bsum[blockIdx.x] = xi;
  }
  __syncthreads();
  if (w < nwords) wprefix[w] = warp_tot[wid] + incl - c;
}

// exclusive scan of the block sums on one CTA
__global__ void __launch_bounds__(kScanBlock) k_bsum_scan(uint32_t* __restrict__ bsum, int64_t nb) {
  __shared__ uint32_t warp_tot[kScanBlock / 32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < nb; base += kScanBlock) {
    const int64_t i = base + threadIdx.x;
    const uint32_t c = i < nb ? bsum[i] : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint32_t x = warp_tot[lane];
      uint32_t xi = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, xi, d);
        if (lane >= d) xi += y;
      }
      warp_tot[lane] = xi - x;
    }
    __syncthreads();
    const uint32_t c0 = carry;
    if (i < nb) bsum[i] = c0 + warp_tot[wid] + incl - c;
    __syncthreads();
    if (threadIdx.x == kScanBlock - 1) carry = c0 + warp_tot[wid] + incl;
    __syncthreads();
  }
}

__device__ __forceinline__ uint32_t bit_rank(uint32_t key, const uint32_t* bitmap,
                                             const uint32_t* wprefix, const uint32_t* bprefix) {
  const uint32_t w = key >> 5;
  return bprefix[w / kScanBlock] + wprefix[w] + __popc(bitmap[w] & ((1u << (key & 31)) - 1u));
}

// sorted[rank(key)] = key, for the pivots
__global__ void k_rank_scatter(const uint32_t* __restrict__ keys, int64_t n,
                               const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ wprefix,
                               const uint32_t* __restrict__ bprefix, uint32_t* __restrict__ sorted) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    sorted[bit_rank(keys[i], bitmap, wprefix, bprefix)] = keys[i];
}

// pivot mask from adjacent bit-reversed keys: lowest differing bit of J
__global__ void k_adjacent_levels(const uint32_t* __restrict__ sorted, int64_t n, int M,
                                  unsigned long long* __restrict__ mask) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = sorted[i - 1] ^ sorted[i];
    const int h = 31 - __clz(x);  // highest differing key bit
    m |= 1ull << (M - 1 - h);
  }
  // warp-reduce then one atomic per warp
  for (int d = 16; d > 0; d >>= 1) m |= __shfl_xor_sync(0xffffffffu, m, d);
  if ((threadIdx.x & 31) == 0 && m) atomicOr(mask, m);
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

// plan-build temporaries come from a library-owned stream-ordered pool that
// keeps its memory (the default pool returns it at every synchronisation, so
// each plan build would re-map its bitmaps and tables from the driver)
static int temp_pool(cudaMemPool_t* pool) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
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
  uint64_t keep = 1024ull << 20;  // keep up to 1 GiB between builds (temporaries and destroyed plans' tables)
  SFFT_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
  pools[dev] = p;
  *pool = p;
  return SFFT_OK;
}

static int alloc(DevBuf& b, size_t bytes, cudaStream_t st) {
  b.st = st;
  cudaMemPool_t pool;
  if (int rc = temp_pool(&pool)) return rc;
  SFFT_CUDA(cudaMallocFromPoolAsync(&b.p, std::max<size_t>(bytes, 16), pool, st));
  return SFFT_OK;
}

// SFFT_PLAN_TRACE=1: synchronise and print the wall time of each plan-build phase (stderr)
struct PlanTrace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0, last;
  explicit PlanTrace(cudaStream_t s) : on(getenv("SFFT_PLAN_TRACE") != nullptr), st(s) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[sfft plan] %-28s %8.3f ms (total %8.3f ms)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(),
            std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

static int grid_1d(int64_t n, int threads = 256) {
  const int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)num_sms() * 16));
}

// Ranks of n distinct keys < 2^L (optionally only those with valid[i]).
struct RankCtx {
  DevBuf bitmap, wprefix, bsum;
  int64_t nwords = 0, nblocks = 0;
};

static int rank_prepare(RankCtx& R, const uint32_t* keys, const uint8_t* valid, int64_t n, int L,
                        cudaStream_t st) {
  R.nwords = std::max<int64_t>(1, (1ll << L) / 32);
  R.nblocks = (R.nwords + kScanBlock - 1) / kScanBlock;
  int rc;
  if ((rc = alloc(R.bitmap, R.nwords * 4, st))) return rc;
  if ((rc = alloc(R.wprefix, R.nwords * 4, st))) return rc;
  if ((rc = alloc(R.bsum, R.nblocks * 4, st))) return rc;
  SFFT_CUDA(cudaMemsetAsync(R.bitmap.p, 0, R.nwords * 4, st));
  if (keys) k_set_bits<<<grid_1d(n), 256, 0, st>>>(keys, valid, n, (uint32_t*)R.bitmap.p);
  return SFFT_OK;
}

static int rank_scan(RankCtx& R, cudaStream_t st) {
  k_word_scan<<<(unsigned)R.nblocks, kScanBlock, 0, st>>>((const uint32_t*)R.bitmap.p, R.nwords,
                                                        (uint32_t*)R.wprefix.p, (uint32_t*)R.bsum.p);
  k_bsum_scan<<<1, kScanBlock, 0, st>>>((uint32_t*)R.bsum.p, R.nblocks);
  SFFT_CUDA(cudaGetLastError());
  return SFFT_OK;
}

static int to_device_J(const int64_t* J, int64_t k, cudaStream_t st, DevBuf& tmp, const int64_t** dJ) {
  if (is_device_pointer(J)) {
    *dJ = J;
    return SFFT_OK;
  }
  int rc = alloc(tmp, sizeof(int64_t) * k, st);
  if (rc) return rc;
  SFFT_CUDA(cudaMemcpyAsync(tmp.p, J, sizeof(int64_t) * k, cudaMemcpyHostToDevice, st));
  *dJ = (const int64_t*)tmp.p;
  return SFFT_OK;
}

// pivots(J) on the device; *mask valid after the call (synchronises)
// O(k) pivots of a homogeneous support (no sort): for homogeneous J every
// pivot is v2(j - j_0), so P0 = OR_e 1 << ctz(J[e] ^ J[0]); J is homogeneous
// with pivots P0 iff |J| = 2^|P0|, j -> pext(j, P0) is a bijection onto the
// 2^|P0| slots, and for every slot x != 0 the elements at x and at x minus
// its top bit first differ exactly at that bit's pivot (then every pairwise
// valuation lies in P0).  Same check as the fused per-signal kernel
// (sfft_fused.cu); a support that fails it takes the general bit-reversed
// rank below.
__global__ void k_homog_mask(const int64_t* __restrict__ J, int64_t k, int M, unsigned long long* __restrict__ w) {
  const int64_t N = 1ll << M;
  unsigned long long m = 0;
  int bad = 0;
  const int64_t j0 = J[0];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = J[e];
    if (j < 0 || j >= N || (e > 0 && J[e - 1] >= j)) bad = 1;
    else if (e > 0) m |= 1ull << __ffsll((unsigned long long)(j ^ j0)) - 1;
  }
  // one atomic per warp (65536 same-address atomics took 45 us on config 5)
  const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)m), hi = __reduce_or_sync(0xffffffffu, (unsigned)(m >> 32));
  const unsigned anybad = __reduce_or_sync(0xffffffffu, (unsigned)bad);
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long mm = ((unsigned long long)hi << 32) | lo;
    if (mm) atomicOr(&w[0], mm);
    if (anybad) atomicOr(&w[1], 1ull);
  }
}
__global__ void k_homog_slots(const int64_t* __restrict__ J, int64_t k, const unsigned long long* __restrict__ w,
                              int32_t* __restrict__ inv, unsigned long long* __restrict__ fail) {
  const unsigned long long P0 = w[0];
  if (w[1] || (1ll << __popcll(P0)) != k) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long j = (unsigned long long)J[e];
    unsigned long long x = 0, m = P0;
    for (int i = 0; m; ++i, m &= m - 1) x |= ((j >> (__ffsll(m) - 1)) & 1ull) << i;
    if (atomicCAS(&inv[x], -1, (int32_t)e) != -1) atomicOr(fail, 1ull);  // two elements, one slot
  }
}
__global__ void k_homog_pairs(const int64_t* __restrict__ J, int64_t k, const unsigned long long* __restrict__ w,
                              const int32_t* __restrict__ inv, unsigned long long* __restrict__ fail) {
  const unsigned long long P0 = w[0];
  if (w[1] || (1ll << __popcll(P0)) != k) return;
  for (int64_t x = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < k; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = 63 - __clzll((unsigned long long)x);
    unsigned long long m = P0;
    for (int i = 0; i < t; ++i) m &= m - 1;
    const int piv = __ffsll(m) - 1;  // pivot of slot bit t
    const int32_t e1 = inv[x], e2 = inv[x ^ (1ll << t)];
    if (e1 < 0 || e2 < 0 || __ffsll((unsigned long long)(J[e1] ^ J[e2])) - 1 != piv) atomicOr(fail, 1ull);
  }
}

static int analyze_device(const int64_t* dJ, int64_t k, int M, uint64_t* mask_out, cudaStream_t st) {
  {  // homogeneous fast path
    DevBuf w, inv;
    int rc;
    if ((rc = alloc(w, 32, st))) return rc;
    SFFT_CUDA(cudaMemsetAsync(w.p, 0, 32, st));
    unsigned long long* dw = (unsigned long long*)w.p;
    const bool pow2 = k > 0 && (k & (k - 1)) == 0 && k <= (1ll << 26);
    if (pow2) {
      if ((rc = alloc(inv, 4 * k, st))) return rc;
      SFFT_CUDA(cudaMemsetAsync(inv.p, 0xff, 4 * k, st));
    }
    k_homog_mask<<<grid_1d(k), 256, 0, st>>>(dJ, k, M, dw);
    if (pow2) {
      k_homog_slots<<<grid_1d(k), 256, 0, st>>>(dJ, k, dw, (int32_t*)inv.p, dw + 2);
      k_homog_pairs<<<grid_1d(k), 256, 0, st>>>(dJ, k, dw, (const int32_t*)inv.p, dw + 2);
    }
    SFFT_CUDA(cudaGetLastError());
    unsigned long long h[3] = {0, 0, 0};
    SFFT_CUDA(cudaMemcpyAsync(h, w.p, 24, cudaMemcpyDeviceToHost, st));
    SFFT_CUDA(cudaStreamSynchronize(st));
    if (h[1]) return fail(SFFT_ERR_INVALID, "support indices must be strictly increasing and lie in [0, N)");
    if (pow2 && h[2] == 0 && (1ll << __builtin_popcountll(h[0])) == k) {
      *mask_out = h[0];
      return SFFT_OK;
    }
    if (k == 1) {
      *mask_out = 0;
      return SFFT_OK;
    }
  }
  DevBuf keys, sorted, small;
  RankCtx R;
  int rc;
  if ((rc = alloc(keys, k * 4, st))) return rc;
  if ((rc = alloc(sorted, k * 4, st))) return rc;
  if ((rc = alloc(small, 16, st))) return rc;
  SFFT_CUDA(cudaMemsetAsync(small.p, 0, 16, st));
  unsigned long long* dmask = (unsigned long long*)small.p;
  int* dstatus = (int*)((char*)small.p + 8);
  if ((rc = rank_prepare(R, nullptr, nullptr, k, M, st))) return rc;
  k_support_keys<<<grid_1d(k), 256, 0, st>>>(dJ, k, M, (uint32_t*)keys.p, (uint32_t*)R.bitmap.p, dstatus);
  if ((rc = rank_scan(R, st))) return rc;
  k_rank_scatter<<<grid_1d(k), 256, 0, st>>>((const uint32_t*)keys.p, k, (const uint32_t*)R.bitmap.p,
                                             (const uint32_t*)R.wprefix.p, (const uint32_t*)R.bsum.p,
                                             (uint32_t*)sorted.p);
  k_adjacent_levels<<<grid_1d(k), 256, 0, st>>>((const uint32_t*)sorted.p, k, M, dmask);
  SFFT_CUDA(cudaGetLastError());
  unsigned long long h[2] = {0, 0};
  SFFT_CUDA(cudaMemcpyAsync(h, small.p, 16, cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  const int status = (int)(h[1] & 0xffffffffu);
  if (status) return fail(SFFT_ERR_INVALID, "support indices must be strictly increasing and lie in [0, N)");
  *mask_out = h[0];
  return SFFT_OK;
}

// --------------------------------------------------------- plan kernels ---
__global__ void k_plan_elements(const int64_t* __restrict__ J, int64_t k, const int32_t* __restrict__ used,
                                int s, int32_t* __restrict__ pats, uint32_t* __restrict__ count,
                                uint32_t* __restrict__ mins, int32_t* __restrict__ inv_elem) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)J[e];
    uint32_t p = 0;
    for (int i = 0; i < s; ++i) p |= ((j >> used[i]) & 1u) << i;
    pats[e] = (int32_t)p;
    atomicAdd(&count[p], 1u);
    atomicMin(&mins[p], j);
    atomicMax(&inv_elem[p], (int32_t)e);  // the one member when mu* = 1
  }
}

// reps level kk (2^kk entries at offset 2^kk - 1) = pairwise min of level kk+1
__global__ void k_min_level(uint32_t* __restrict__ reps, int kk) {
  const int64_t n = 1ll << kk;
  uint32_t* lo = reps + (n - 1);
  const uint32_t* hi = reps + (2 * n - 1);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    lo[x] = min(hi[x], hi[x + n]);
}

// empty prefixes inherit parent residue below r with the branch bit set (hidft.py:87-90)
__global__ void k_fill_level(uint32_t* __restrict__ reps, int kk, int r) {
  const int64_t n = 1ll << kk;
  uint32_t* cur = reps + (n - 1);
  const uint32_t* par = reps + (n / 2 - 1);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (cur[x] != 0xffffffffu) continue;
    const uint32_t shared = par[x & (n / 2 - 1)] & ((1u << r) - 1u);
    cur[x] = shared + ((uint32_t)((x >> (kk - 1)) & 1) << r);
  }
}

// levels kk = top .. 0 of k_min_level in one CTA (2^top <= 4096 entries)
__global__ void __launch_bounds__(1024) k_min_levels_cta(uint32_t* __restrict__ reps, int top) {
  for (int kk = top; kk >= 0; --kk) {
    const int n = 1 << kk;
    for (int x = threadIdx.x; x < n; x += blockDim.x) reps[n - 1 + x] = min(reps[2 * n - 1 + x], reps[3 * n - 1 + x]);
    __syncthreads();
  }
}
// levels kk = 1 .. top of k_fill_level in one CTA
__global__ void __launch_bounds__(1024) k_fill_levels_cta(uint32_t* __restrict__ reps, int top,
                                                          const int32_t* __restrict__ used) {
  for (int kk = 1; kk <= top; ++kk) {
    const int n = 1 << kk, r = used[kk - 1];
    for (int x = threadIdx.x; x < n; x += blockDim.x) {
      uint32_t* cur = reps + (n - 1);
      if (cur[x] != 0xffffffffu) continue;
      const uint32_t shared = reps[n / 2 - 1 + (x & (n / 2 - 1))] & ((1u << r) - 1u);
      cur[x] = shared + ((uint32_t)((x >> (kk - 1)) & 1) << r);
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void k_plan_twiddles(const uint32_t* __restrict__ reps, const int32_t* __restrict__ used,
                                int64_t A, Cx<T>* __restrict__ tw) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < A - 1;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int beta = 63 - __clzll(idx + 1);
    const int64_t h = idx + 1 - (1ll << beta);
    const int rk = used[beta];
    const uint32_t shared = reps[(1ll << beta) - 1 + h] & ((1u << rk) - 1u);
    double c, s;
    twiddle_d(shared, rk, c, s);
    tw[idx] = Cx<T>{(T)c, (T)s};
  }
}

__global__ void k_plan_slots(const uint32_t* __restrict__ reps_s, const uint32_t* __restrict__ count,
                             int64_t A, int level, int32_t* __restrict__ slot_res,
                             uint8_t* __restrict__ slot_real, unsigned long long* __restrict__ stats) {
  const uint32_t lmask = level >= 32 ? 0xffffffffu : ((1u << level) - 1u);
  unsigned long long nreal = 0, mu = 0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < A;
       x += (int64_t)gridDim.x * blockDim.x) {
    slot_res[x] = (int32_t)(reps_s[x] & lmask);
    const uint32_t c = count[x];
    slot_real[x] = c > 0;
    nreal += c > 0;
    mu = mu > c ? mu : c;
  }
  for (int d = 16; d > 0; d >>= 1) {
    nreal += __shfl_xor_sync(0xffffffffu, nreal, d);
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, mu, d);
    mu = mu > o ? mu : o;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&stats[0], nreal);
    atomicMax(&stats[1], mu);
  }
}

__global__ void k_node_order(const int32_t* __restrict__ slot_res, const uint8_t* __restrict__ slot_real,
                             int64_t A, const uint32_t* __restrict__ bitmap,
                             const uint32_t* __restrict__ wprefix, const uint32_t* __restrict__ bprefix,
                             int32_t* __restrict__ node_slots, int32_t* __restrict__ node_res,
                             int32_t* __restrict__ inv_node) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < A;
       x += (int64_t)gridDim.x * blockDim.x) {
    if (!slot_real[x]) continue;
    const uint32_t res = (uint32_t)slot_res[x];
    const uint32_t rk = bit_rank(res, bitmap, wprefix, bprefix);
    node_slots[rk] = (int32_t)x;
    node_res[rk] = (int32_t)res;
    inv_node[x] = (int32_t)rk;
  }
}

__global__ void k_node_identity(const int64_t* __restrict__ J, int64_t k, const int32_t* __restrict__ pats,
                                int32_t* __restrict__ node_slots, int32_t* __restrict__ node_res,
                                int32_t* __restrict__ inv_node) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    node_slots[e] = pats[e];
    node_res[e] = (int32_t)J[e];
    inv_node[pats[e]] = (int32_t)e;
  }
}

__global__ void k_offsets(const int32_t* __restrict__ used, int s, int M, int64_t A, int64_t* __restrict__ off,
                          int sorted_order) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < A;
       a += (int64_t)gridDim.x * blockDim.x) {
    // slot order: off(a) = sum_i bit_i(a) 2^(M-1-used_i) (hidft.py:155-158);
    // sorted order (I_r ascending) is the same sum over the bit-reversed index.
    int64_t v = 0;
    for (int i = 0; i < s; ++i) {
      const int bit = sorted_order ? (int)((a >> (s - 1 - i)) & 1) : (int)((a >> i) & 1);
      v += (int64_t)bit << (M - 1 - used[i]);
    }
    off[a] = v;
  }
}

__global__ void k_widen(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

}  // namespace sfft

// ------------------------------------------------------------------ C-ABI ---
using namespace sfft;

static int validate_r(const int32_t* r, int n_r, int M) {
  if (n_r < 0 || n_r > 31) return fail(SFFT_ERR_INVALID, "pivot vector too long");
  if (n_r > 0 && !r) return fail(SFFT_ERR_INVALID, "null pivot vector");
  for (int i = 0; i + 1 < n_r; ++i)
    if (r[i] >= r[i + 1]) return fail(SFFT_ERR_INVALID, "pivot vector must be strictly increasing");
  for (int i = 0; i < n_r; ++i)
    if (r[i] < 0 || r[i] >= M)
      return fail(SFFT_ERR_INVALID, "pivots must lie in [0, " + std::to_string(M) + ")");
  return SFFT_OK;
}

static std::string tuple_str(const int32_t* r, int n) {
  std::string s = "(";
  for (int i = 0; i < n; ++i) s += std::to_string(r[i]) + (n == 1 ? "," : (i + 1 < n ? ", " : ""));
  return s + ")";
}

extern "C" const char* sfft_version(void) { return "structfft_b200 0.1.0 (sm_100a)"; }
extern "C" const char* sfft_last_error(void) { return g_last_error.c_str(); }

extern "C" int sfft_device_ok(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

extern "C" int sfft_analyze(const int64_t* J, int64_t k, int M, uint64_t* pivot_mask, int* homogeneous,
                            sfft_stream_t stream) {
  SFFT_NVTX("sfft_analyze");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (!J) return fail(SFFT_ERR_INVALID, "null support");
  DevBuf tmp;
  const int64_t* dJ = nullptr;
  int rc = to_device_J(J, k, st, tmp, &dJ);
  if (rc) return rc;
  uint64_t mask = 0;
  if ((rc = analyze_device(dJ, k, M, &mask, st))) return rc;
  if (pivot_mask) *pivot_mask = mask;
  if (homogeneous) *homogeneous = (k & (k - 1)) == 0 && __builtin_popcountll(mask) == 63 - __builtin_clzll(k);
  return SFFT_OK;
}

__global__ void k_pattern(const int32_t* __restrict__ r, int n, int M, int64_t* __restrict__ out) {
  const int64_t A = 1ll << n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < A;
       q += (int64_t)gridDim.x * blockDim.x) {
    // bit j of q (ascending) carries pivot r[n-1-j]: smallest offsets first
    int64_t v = 0;
    for (int j = 0; j < n; ++j) v += ((q >> j) & 1) << (M - 1 - r[n - 1 - j]);
    out[q] = v;
  }
}

extern "C" int sfft_pivoted_pattern(const int32_t* r, int n_r, int M, int64_t* out, sfft_stream_t stream) {
  SFFT_NVTX("sfft_pivoted_pattern");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 62) return fail(SFFT_ERR_INVALID, "M out of range");
  int rc = validate_r(r, n_r, M);
  if (rc) return rc;
  if (n_r > 30) return fail(SFFT_ERR_UNSUPPORTED, "pattern too large");
  const int64_t A = 1ll << n_r;
  DevBuf dr, dout;
  if ((rc = alloc(dr, sizeof(int32_t) * std::max(n_r, 1), st))) return rc;
  if (n_r) SFFT_CUDA(cudaMemcpyAsync(dr.p, r, sizeof(int32_t) * n_r, cudaMemcpyHostToDevice, st));
  const bool dev_out = is_device_pointer(out);
  int64_t* target = out;
  if (!dev_out) {
    if ((rc = alloc(dout, sizeof(int64_t) * A, st))) return rc;
    target = (int64_t*)dout.p;
  }
  k_pattern<<<grid_1d(A), 256, 0, st>>>((const int32_t*)dr.p, n_r, M, target);
  SFFT_CUDA(cudaGetLastError());
  if (!dev_out) {
    SFFT_CUDA(cudaMemcpyAsync(out, target, sizeof(int64_t) * A, cudaMemcpyDeviceToHost, st));
    SFFT_CUDA(cudaStreamSynchronize(st));
  }
  return SFFT_OK;
}

// Block-major tables of the split transform: block t (2^lc of them) holds the
// slots a = (l << lc) | brev_lc(t); its local stage k' (global stage lc + k')
// twiddle h' is tw_{lc+k'}[(h' << lc) | brev_lc(t)] (hidft.py:160-167).
template <typename T>
__global__ void k_split_tables(const Cx<T>* __restrict__ tw, const int32_t* __restrict__ inv_elem,
                               const int32_t* __restrict__ inv_node, int s, int lc, Cx<T>* __restrict__ tw_blk,
                               int32_t* __restrict__ inv_elem_blk, int32_t* __restrict__ inv_node_blk) {
  const int sl = s - lc;
  const int64_t A = 1ll << s, AL = 1ll << sl;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i >> sl), l = (uint32_t)(i & (AL - 1));
    const uint32_t low = lc ? (__brev(t) >> (32 - lc)) : 0u;
    const uint32_t a = (l << lc) | low;
    inv_elem_blk[i] = inv_elem[a];
    inv_node_blk[i] = inv_node[a];
    if (l + 1 < AL) {  // local stage-major index m = l: stage k' = floor(log2(m+1)) + 1
      const int kp = 32 - __clz(l + 1);
      const uint32_t hp = l + 1 - (1u << (kp - 1));
      const int k = lc + kp;
      tw_blk[(int64_t)t * (AL - 1) + l] = tw[((int64_t)1 << (k - 1)) - 1 + ((hp << lc) | low)];
    }
  }
}

// Three-pass split (sfft_split.cu, k_tri_*).  Slot a = (b << (s-4)) | q: the
// final pass runs the last 4 stages (pairing b's bits) for a fixed q, so its
// 16 results land at inv[(b << (s-4)) | q].  When the top 4 pivots are the top
// 4 bits of j (config 5), j = b*2^(M-4) + h(q) and the output position is
// b*2^(s-4) + sigma(q): ordering q by its mean output position (the key
// below) makes every final-pass store run contiguous.  Other supports get the
// same ordering as a heuristic (correctness never depends on it).
__global__ void k_tri_key(const int32_t* __restrict__ inv, int s, int64_t n_out, double* __restrict__ key) {
  const int sq = s - 4;
  const int64_t nq = 1ll << sq;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double per_b = (double)n_out / 16.0;
  double sum = 0.0;
  int cnt = 0;
  for (int b = 0; b < 16; ++b) {
    const int32_t v = inv[((int64_t)b << sq) | q];
    if (v >= 0) {
      sum += (double)v - b * per_b;
      ++cnt;
    }
  }
  key[q] = cnt ? sum / cnt : 1e18 + (double)q;
}

// perm[rank(q)] = q, rank by (key, q): one CTA bitonic-sorts the (key, q)
// pairs in shared memory (nq <= 8192: 96 KB), O(nq log^2 nq) compares
// instead of the O(nq^2) all-pairs rank.
__global__ void __launch_bounds__(1024) k_tri_sort(const double* __restrict__ key, int nq,
                                                   int32_t* __restrict__ perm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sk = reinterpret_cast<double*>(smem_raw);
  int32_t* sq = reinterpret_cast<int32_t*>(sk + nq);
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    sk[i] = key[i];
    sq[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= nq; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < nq; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const double ki = sk[i], kj = sk[j];
          const int32_t qi = sq[i], qj = sq[j];
          const bool gt = ki > kj || (ki == kj && qi > qj);
          if (gt == up) {
            sk[i] = kj;
            sk[j] = ki;
            sq[i] = qj;
            sq[j] = qi;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < nq; i += blockDim.x) perm[i] = sq[i];
}

// The same order by a parallel rank: every thread counts the (key, q) pairs
// below its own among all nq keys staged in shared memory (broadcast reads),
// nq / 128 CTAs; 4096 keys: ~8 us against 62 us for the one-CTA sort.
__global__ void __launch_bounds__(128) k_tri_rank(const double* __restrict__ key, int nq, int32_t* __restrict__ perm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sk = reinterpret_cast<double*>(smem_raw);
  for (int i = threadIdx.x; i < nq; i += blockDim.x) sk[i] = key[i];
  __syncthreads();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double kq = sk[q];
  int rank = 0;
#pragma unroll 8
  for (int i = 0; i < nq; ++i) {
    const double ki = sk[i];
    rank += (ki < kq || (ki == kq && i < q)) ? 1 : 0;
  }
  perm[rank] = q;
}

// blocked output map of the final pass (k_fin2): inv[b][pi] = T * nq + pi
// for every b, pi; flag stays 1 only if all entries comply
__global__ void k_blocked_check(const int32_t* __restrict__ inv, int64_t A, int64_t nq,
                                unsigned long long* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = inv[i];
    if (v < 0 || (v & (nq - 1)) != (i & (nq - 1))) atomicAnd(flag, 0ull);
  }
}

// Final-pass tables in pi order: stage s-4+t (t < 4) pairs slot bit s-4+t
// with twiddle index a mod 2^(s-4+t) = q | (c << (s-4)), c = b mod 2^t
// (hidft.py:160-167); j = 2^t - 1 + c.
template <typename T>
__global__ void k_tri_tables(const Cx<T>* __restrict__ tw, const int32_t* __restrict__ inv_elem,
                             const int32_t* __restrict__ inv_node, const int32_t* __restrict__ perm, int s,
                             Cx<T>* __restrict__ tw_fin, int32_t* __restrict__ inv_elem_fin,
                             int32_t* __restrict__ inv_node_fin, int32_t* __restrict__ pinv) {
  const int sq = s - 4;
  const int64_t nq = 1ll << sq;
  const int64_t pi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (pi >= nq) return;
  const int64_t q = perm[pi];
  pinv[q] = (int32_t)pi;
  for (int b = 0; b < 16; ++b) {
    inv_elem_fin[b * nq + pi] = inv_elem[((int64_t)b << sq) | q];
    inv_node_fin[b * nq + pi] = inv_node[((int64_t)b << sq) | q];
  }
  for (int t = 0; t < 4; ++t)
    for (int c = 0; c < (1 << t); ++c)
      tw_fin[((1 << t) - 1 + c) * nq + pi] = tw[((int64_t)1 << (sq + t)) - 1 + (q | ((int64_t)c << sq))];
}

// Bank-conflict-free layout for the complex64 middle pass (sfft_split.cu,
// k_tri_mid).  Its last register pass stores one value per lane per warp
// instruction (group "store": a half-warp's 16 lanes for register x) and its
// epilogue reads consecutive pi, i.e. q = perm[pi] (group "read": 16
// consecutive pi).  8 B accesses are served per half-warp, conflict-free
// when its 16 lanes hit the 16 word slots (position mod 16) once each.  The
// q's form a 16-regular bipartite multigraph between store groups and read
// groups (edge q); four Euler splits (alternate the edges of closed trails:
// every vertex keeps half its edges on each side) cut it into 16 perfect
// matchings, and matching c becomes word slot c: position = 16 * (rank of q
// within class c) + c.  Host code, once per plan.
static void euler_split(const std::vector<int>& edges, const std::vector<int>& eu, const std::vector<int>& ev,
                        int nv, std::vector<int>& A, std::vector<int>& B) {
  // vertices 0..nv-1 (stores) and nv..2nv-1 (reads)
  std::vector<std::vector<int>> adj(2 * nv);
  for (int e : edges) {
    adj[eu[e]].push_back(e);
    adj[nv + ev[e]].push_back(e);
  }
  std::vector<char> used(eu.size(), 0);
  std::vector<size_t> ptr(2 * nv, 0);
  for (int start = 0; start < 2 * nv; ++start) {
    for (;;) {
      while (ptr[start] < adj[start].size() && used[adj[start][ptr[start]]]) ++ptr[start];
      if (ptr[start] == adj[start].size()) break;
      // closed trail from start, labels alternate A, B, A, ...
      int v = start, side = 0;
      for (;;) {
        while (ptr[v] < adj[v].size() && used[adj[v][ptr[v]]]) ++ptr[v];
        if (ptr[v] == adj[v].size()) break;  // back at start with nothing left (degrees are even)
        const int e = adj[v][ptr[v]];
        used[e] = 1;
        (side ? B : A).push_back(e);
        side ^= 1;
        v = (v < nv) ? nv + ev[e] : eu[e];
      }
    }
  }
}

// Conflict-free word slots for one store/read pattern: edge e = (store group
// eu[e], read group ev[e]) is the value q = qof[e]; both groupings are
// 16-regular over NQ/16 groups.  Four Euler splits cut the edges into 16
// perfect matchings; matching c is word slot c: posq[q] = 16 * (rank of q
// in its class) + c.  False when a split is unbalanced (keep the swizzle).
static bool conflict_free_positions(const std::vector<int>& eu, const std::vector<int>& ev,
                                    const std::vector<int>& qof, int NQ, std::vector<int32_t>& posq) {
  const int nv = NQ / 16;
  std::vector<std::vector<int>> cls(1);
  cls[0].resize(NQ);
  for (int e = 0; e < NQ; ++e) cls[0][e] = e;
  for (int lvl = 0; lvl < 4; ++lvl) {
    std::vector<std::vector<int>> next;
    for (auto& c : cls) {
      std::vector<int> A, B;
      euler_split(c, eu, ev, nv, A, B);
      next.push_back(std::move(A));
      next.push_back(std::move(B));
    }
    cls.swap(next);
  }
  posq.assign(NQ, -1);
  for (int c = 0; c < 16; ++c) {
    if ((int)cls[c].size() != NQ / 16) return false;
    for (int r = 0; r < (int)cls[c].size(); ++r) posq[qof[cls[c][r]]] = 16 * r + c;
  }
  std::vector<char> seen(NQ, 0);
  for (int q = 0; q < NQ; ++q) {
    if (posq[q] < 0 || posq[q] >= NQ || seen[posq[q]]) return false;
    seen[posq[q]] = 1;
  }
  // every store and read group hits each word slot once
  std::vector<int> cs((size_t)nv * 16, 0), cr((size_t)nv * 16, 0);
  for (int e = 0; e < NQ; ++e) {
    if (++cs[(size_t)eu[e] * 16 + (posq[qof[e]] & 15)] > 1) return false;
    if (++cr[(size_t)ev[e] * 16 + (posq[qof[e]] & 15)] > 1) return false;
  }
  return true;
}

static int upload_tables(const std::vector<int32_t>& a, const std::vector<int32_t>& b, int32_t** da, int32_t** db) {
  int32_t* x = nullptr;
  int32_t* y = nullptr;
  SFFT_CUDA(cudaMalloc((void**)&x, 4 * a.size()));
  if (cudaMalloc((void**)&y, 4 * b.size()) != cudaSuccess) {
    cudaFree(x);
    return cuda_fail(cudaGetLastError(), "conflict-free table allocation");
  }
  const cudaError_t e1 = cudaMemcpy(x, a.data(), 4 * a.size(), cudaMemcpyHostToDevice);
  const cudaError_t e2 = cudaMemcpy(y, b.data(), 4 * b.size(), cudaMemcpyHostToDevice);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaFree(x);
    cudaFree(y);
    return cuda_fail(e1 != cudaSuccess ? e1 : e2, "conflict-free table upload");
  }
  *da = x;
  *db = y;
  return SFFT_OK;
}

static int tri_conflict_free_tables(sfft_plan* p, cudaStream_t st) {
  const int s = p->s;
  const int F = s == 15 ? 3 : 4, L = 4, MID = s - F - L, SQ = s - L;
  const int NQ = 1 << SQ, EX = 1 << F, LE = 4, E2 = std::min(16, 1 << MID), NT = NQ / E2;
  const int NPASS = (MID + LE - 1) / LE, last = NPASS - 1;
  if (MID < LE || NQ % 32 || NT % 32) return SFFT_OK;
  std::vector<int32_t> perm(NQ), pinv(NQ);
  SFFT_CUDA(cudaMemcpyAsync(perm.data(), p->d_tri_perm, 4 * (size_t)NQ, cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  for (int pi = 0; pi < NQ; ++pi) pinv[perm[pi]] = pi;
  // q stored by thread tid from register x in the last pass (k_tri_mid: a = tid & (EX-1), mr = tid >> F)
  const int w0 = (last * LE < MID - LE) ? last * LE : MID - LE;
  std::vector<int> eu(NQ), ev(NQ), qof(NQ);  // edge index = x * NT + tid
  for (int x = 0; x < E2; ++x)
    for (int tid = 0; tid < NT; ++tid) {
      const int a = tid & (EX - 1), mr = tid >> F;
      const int slot = (mr & ((1 << w0) - 1)) | ((mr >> w0) << (w0 + LE)) | (x << w0);
      const int q = (slot << F) | a;
      const int e = x * NT + tid;
      qof[e] = q;
      eu[e] = (tid >> 4) * E2 + x;  // store group: a half-warp's lanes for register x
      ev[e] = pinv[q] >> 4;         // read group: 16 consecutive pi
    }
  std::vector<int32_t> posq;
  if (!conflict_free_positions(eu, ev, qof, NQ, posq)) return SFFT_OK;  // keep the swizzled layout
  std::vector<int32_t> spos(NQ), ppos(NQ);
  for (int e = 0; e < NQ; ++e) spos[e] = posq[qof[e]];
  for (int pi = 0; pi < NQ; ++pi) ppos[pi] = posq[perm[pi]];
  return upload_tables(spos, ppos, &p->d_tri_spos, &p->d_tri_ppos);
}

// The head pass (sfft_split.cu, k_head) in the same way: its last register
// pass stores slot(tt, x) from thread tt's register x (a half-warp: 16
// consecutive tt, fixed x), its epilogue reads pi = tt + n * 2^(SQ-4), q =
// perm[pi] (a half-warp: 16 consecutive pi).  Tables: spos[x * TPB + tt],
// ppos[pi], positions inside one b value's 2^SQ-slot block.
static int head_conflict_free_tables(sfft_plan* p, cudaStream_t st) {
  const int SQ = p->s - 4, NQ = 1 << SQ, LE = 4, E = 16, TPB = NQ / E;
  const int NPASS = (SQ + LE - 1) / LE, last = NPASS - 1;
  const int w0 = (last * LE < SQ - LE) ? last * LE : SQ - LE;
  if (TPB % 16) return SFFT_OK;
  std::vector<int32_t> perm(NQ), pinv(NQ);
  SFFT_CUDA(cudaMemcpyAsync(perm.data(), p->d_tri_perm, 4 * (size_t)NQ, cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  for (int pi = 0; pi < NQ; ++pi) pinv[perm[pi]] = pi;
  std::vector<int> eu(NQ), ev(NQ), qof(NQ);  // edge index = x * TPB + tt
  for (int x = 0; x < E; ++x)
    for (int tt = 0; tt < TPB; ++tt) {
      const int q = (tt & ((1 << w0) - 1)) | ((tt >> w0) << (w0 + LE)) | (x << w0);
      const int e = x * TPB + tt;
      qof[e] = q;
      eu[e] = x * (TPB / 16) + (tt >> 4);
      ev[e] = pinv[q] >> 4;
    }
  std::vector<int32_t> posq;
  if (!conflict_free_positions(eu, ev, qof, NQ, posq)) return SFFT_OK;
  std::vector<int32_t> spos(NQ), ppos(NQ);
  for (int e = 0; e < NQ; ++e) spos[e] = posq[qof[e]];
  for (int pi = 0; pi < NQ; ++pi) ppos[pi] = posq[perm[pi]];
  return upload_tables(spos, ppos, &p->d_head_spos, &p->d_head_ppos);
}

static void plan_free(sfft_plan* p) {
  if (!p) return;
  cudaFree(p->d_element_slots);
  cudaFree(p->d_slot_residues);
  cudaFree(p->d_slot_real);
  cudaFree(p->d_node_slots);
  cudaFree(p->d_node_residues);
  cudaFree(p->d_twiddles);
  cudaFree(p->d_inv_elem);
  cudaFree(p->d_inv_node);
  cudaFree(p->d_node_off);
  cudaFree(p->d_node_mem);
  cudaFree(p->d_node_x);
  cudaFree(p->d_node_perm);
  cudaFree(p->d_node_amp);
  cudaFree(p->d_tw_blk);
  cudaFree(p->d_inv_elem_blk);
  cudaFree(p->d_inv_node_blk);
  cudaFree(p->d_tri_perm);
  cudaFree(p->d_tri_pinv);
  cudaFree(p->d_tri_tw);
  cudaFree(p->d_tri_inv_elem);
  cudaFree(p->d_tri_inv_node);
  cudaFree(p->d_tri_spos);
  cudaFree(p->d_tri_ppos);
  cudaFree(p->d_head_spos);
  cudaFree(p->d_head_ppos);
  cudaFree(p->d_J);
  delete p;
}

extern "C" int sfft_plan_create(const int64_t* J, int64_t k, int M, const int32_t* r, int n_r, int height,
                                int dtype, sfft_stream_t stream, sfft_plan** out_plan) {
  SFFT_NVTX("sfft_plan_create");
  cudaStream_t st = (cudaStream_t)stream;
  if (!out_plan) return fail(SFFT_ERR_INVALID, "null plan output");
  *out_plan = nullptr;
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (dtype != SFFT_C64 && dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown dtype");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  int rc = validate_r(r, n_r, M);  // congruence.py:272-278
  if (rc) return rc;
  PlanTrace trace(st);
  DevBuf tmpJ;
  const int64_t* dJ = nullptr;
  if ((rc = to_device_J(J, k, st, tmpJ, &dJ))) return rc;
  uint64_t mask = 0;
  trace.mark("support upload");
  if ((rc = analyze_device(dJ, k, M, &mask, st))) return rc;
  trace.mark("analyze (pivots)");
  if (n_r > 0) {  // assert_part_homogeneous, congruence.py:259-269
    const int rmax = r[n_r - 1];
    uint64_t rmask = 0;
    for (int i = 0; i < n_r; ++i) rmask |= 1ull << r[i];
    const uint64_t bad = mask & ((2ull << rmax) - 1) & ~rmask;
    if (bad)
      return fail(SFFT_ERR_CONTRACT, "support is not " + tuple_str(r, n_r) + "-part-homogeneous: pivot " +
                                         std::to_string(__builtin_ctzll(bad)) + " <= " + std::to_string(rmax) +
                                         " missing from r");
  }
  if (height < 0 || height > n_r)
    return fail(SFFT_ERR_INVALID, "height must be in [0, " + std::to_string(n_r) + "]");
  const int s = n_r - height;
  if (s > 26) return fail(SFFT_ERR_UNSUPPORTED, "more than 2^26 slots");
  const int64_t A = 1ll << s;
  const int level = s ? r[s - 1] + 1 : 0;

  sfft_plan* p = new sfft_plan();
  std::memset(p, 0, sizeof(*p));
  SFFT_CUDA(cudaGetDevice(&p->device));
  p->M = M;
  p->dtype = dtype;
  p->n_r = n_r;
  p->height = height;
  p->s = s;
  p->level = level;
  p->k = k;
  p->A = A;
  p->pivot_mask = mask;
  p->homogeneous = (k & (k - 1)) == 0 && __builtin_popcountll(mask) == 63 - __builtin_clzll(k);
  for (int i = 0; i < n_r; ++i) p->r[i] = r[i];
  for (int i = 0; i < s; ++i) p->used[i] = r[i];
  const size_t csz = dtype == SFFT_C64 ? 8 : 16;
  cudaError_t e = cudaSuccess;
  // the plan's tables come from the library's stream-ordered pool as well
  // (a destroyed plan's memory serves the next build without a driver
  // allocation per table; plan_free releases them with cudaFree, which
  // synchronises as before)
  cudaMemPool_t tpool;
  if (int prc = temp_pool(&tpool)) {
    delete p;
    return prc;
  }
  auto M_ = [&](void** ptr, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(ptr, std::max<size_t>(bytes, 16), tpool, st);
  };
  M_((void**)&p->d_element_slots, 4 * k);
  M_((void**)&p->d_slot_residues, 4 * A);
  M_((void**)&p->d_slot_real, A);
  M_((void**)&p->d_node_slots, 4 * std::min<int64_t>(A, k));
  M_((void**)&p->d_node_residues, 4 * std::min<int64_t>(A, k));
  M_(&p->d_twiddles, csz * std::max<int64_t>(A - 1, 1));
  M_((void**)&p->d_inv_elem, 4 * A);
  M_((void**)&p->d_inv_node, 4 * A);
  if (e != cudaSuccess) {
    plan_free(p);
    return cuda_fail(e, "plan allocation");
  }
  auto done = [&](int code) {
    if (code) plan_free(p);
    return code;
  };
  DevBuf dused, count, reps, stats;
  if ((rc = alloc(dused, 4 * 32, st))) return done(rc);
  if ((rc = alloc(count, 4 * A, st))) return done(rc);
  if ((rc = alloc(reps, 4 * (2 * A - 1), st))) return done(rc);
  if ((rc = alloc(stats, 32, st))) return done(rc);
  if (cudaMemcpyAsync(dused.p, p->used, 4 * 32, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(count.p, 0, 4 * A, st) != cudaSuccess ||
      cudaMemsetAsync(reps.p, 0xff, 4 * (2 * A - 1), st) != cudaSuccess ||
      cudaMemsetAsync(stats.p, 0, 16, st) != cudaSuccess ||
      cudaMemsetAsync((char*)stats.p + 16, 0xff, 16, st) != cudaSuccess ||
      cudaMemsetAsync(p->d_inv_elem, 0xff, 4 * A, st) != cudaSuccess ||
      cudaMemsetAsync(p->d_inv_node, 0xff, 4 * A, st) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "plan init"));
  uint32_t* dreps = (uint32_t*)reps.p;
  const int32_t* du = (const int32_t*)dused.p;
  k_plan_elements<<<grid_1d(k), 256, 0, st>>>(dJ, k, du, s, p->d_element_slots, (uint32_t*)count.p,
                                              dreps + (A - 1), p->d_inv_elem);
  constexpr int kCtaLevels = 12;  // levels of <= 4096 entries run in one CTA launch
  for (int kk = s - 1; kk >= kCtaLevels; --kk) k_min_level<<<grid_1d(1ll << kk), 256, 0, st>>>(dreps, kk);
  if (s > 0) k_min_levels_cta<<<1, 1024, 0, st>>>(dreps, std::min(s - 1, kCtaLevels - 1));
  if (s > 0) k_fill_levels_cta<<<1, 1024, 0, st>>>(dreps, std::min(s, kCtaLevels), du);
  for (int kk = kCtaLevels + 1; kk <= s; ++kk)
    k_fill_level<<<grid_1d(1ll << kk), 256, 0, st>>>(dreps, kk, p->used[kk - 1]);
  if (A > 1) {
    if (dtype == SFFT_C64)
      k_plan_twiddles<float><<<grid_1d(A), 256, 0, st>>>(dreps, du, A, (Cx<float>*)p->d_twiddles);
    else
      k_plan_twiddles<double><<<grid_1d(A), 256, 0, st>>>(dreps, du, A, (Cx<double>*)p->d_twiddles);
  }
  k_plan_slots<<<grid_1d(A), 256, 0, st>>>(dreps + (A - 1), (const uint32_t*)count.p, A, level,
                                           p->d_slot_residues, p->d_slot_real,
                                           (unsigned long long*)stats.p);
  if (p->homogeneous && height == 0 && level == M && k == A) {
    // every slot is real and its residue mod 2^M is its element: ascending
    // residue is J's own (sorted) order, no rank over 2^M bits needed
    k_node_identity<<<grid_1d(k), 256, 0, st>>>(dJ, k, p->d_element_slots, p->d_node_slots, p->d_node_residues,
                                                p->d_inv_node);
  } else {
    RankCtx R;
    if ((rc = rank_prepare(R, nullptr, nullptr, A, level, st))) return done(rc);
    // residues of real slots are distinct: set their bits, then rank
    k_set_bits<<<grid_1d(A), 256, 0, st>>>((const uint32_t*)p->d_slot_residues, p->d_slot_real, A,
                                           (uint32_t*)R.bitmap.p);
    if ((rc = rank_scan(R, st))) return done(rc);
    k_node_order<<<grid_1d(A), 256, 0, st>>>(p->d_slot_residues, p->d_slot_real, A,
                                             (const uint32_t*)R.bitmap.p, (const uint32_t*)R.wprefix.p,
                                             (const uint32_t*)R.bsum.p, p->d_node_slots, p->d_node_residues,
                                             p->d_inv_node);
  }
  trace.mark("slots, twiddles, node order");
  p->split_lc = split_lc(dtype, s);
  if (p->split_lc) {
    if (split_two_pass()) {  // block-major tables of the two-pass transform (k_split_*, SFFT_SPLIT_PASSES=2)
      const int lc = p->split_lc, sl = s - lc;
      M_(&p->d_tw_blk, csz * ((size_t)1 << lc) * (((size_t)1 << sl) - 1));
      M_((void**)&p->d_inv_elem_blk, 4 * A);
      M_((void**)&p->d_inv_node_blk, 4 * A);
      if (e != cudaSuccess) return done(cuda_fail(e, "split table allocation"));
      if (dtype == SFFT_C64)
        k_split_tables<float><<<grid_1d(A), 256, 0, st>>>((const Cx<float>*)p->d_twiddles, p->d_inv_elem,
                                                          p->d_inv_node, s, lc, (Cx<float>*)p->d_tw_blk,
                                                          p->d_inv_elem_blk, p->d_inv_node_blk);
      else
        k_split_tables<double><<<grid_1d(A), 256, 0, st>>>((const Cx<double>*)p->d_twiddles, p->d_inv_elem,
                                                           p->d_inv_node, s, lc, (Cx<double>*)p->d_tw_blk,
                                                           p->d_inv_elem_blk, p->d_inv_node_blk);
    }
    // three-pass tables (k_tri_*)
    const int64_t nq = A >> 4;
    M_((void**)&p->d_tri_perm, 4 * nq);
    M_((void**)&p->d_tri_pinv, 4 * nq);
    M_(&p->d_tri_tw, csz * 15 * nq);
    M_((void**)&p->d_tri_inv_elem, 4 * A);
    M_((void**)&p->d_tri_inv_node, 4 * A);
    DevBuf key;
    if (e != cudaSuccess) return done(cuda_fail(e, "split table allocation"));
    if ((rc = alloc(key, 8 * nq, st))) return done(rc);
    k_tri_key<<<grid_1d(nq), 256, 0, st>>>(p->homogeneous ? p->d_inv_elem : p->d_inv_node, s,
                                            p->homogeneous ? k : std::min<int64_t>(A, k), (double*)key.p);
    if (nq >= 128 && nq <= 16384) {  // parallel rank (keys fit one CTA's shared memory)
      const size_t sm = (size_t)nq * sizeof(double);
      if (cudaFuncSetAttribute(k_tri_rank, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return done(cuda_fail(cudaGetLastError(), "plan rank"));
      k_tri_rank<<<(unsigned)(nq / 128), 128, sm, st>>>((const double*)key.p, (int)nq, p->d_tri_perm);
    } else {
      const size_t sm = (size_t)nq * (sizeof(double) + sizeof(int32_t));
      if (cudaFuncSetAttribute(k_tri_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return done(cuda_fail(cudaGetLastError(), "plan sort"));
      k_tri_sort<<<1, 1024, sm, st>>>((const double*)key.p, (int)nq, p->d_tri_perm);
    }
    if (dtype == SFFT_C64)
      k_tri_tables<float><<<grid_1d(nq), 256, 0, st>>>((const Cx<float>*)p->d_twiddles, p->d_inv_elem,
                                                        p->d_inv_node, p->d_tri_perm, s, (Cx<float>*)p->d_tri_tw,
                                                        p->d_tri_inv_elem, p->d_tri_inv_node, p->d_tri_pinv);
    else
      k_tri_tables<double><<<grid_1d(nq), 256, 0, st>>>((const Cx<double>*)p->d_twiddles, p->d_inv_elem,
                                                         p->d_inv_node, p->d_tri_perm, s,
                                                         (Cx<double>*)p->d_tri_tw, p->d_tri_inv_elem,
                                                         p->d_tri_inv_node, p->d_tri_pinv);
  }
  trace.mark("split / three-pass tables");
  unsigned long long h[4] = {0, 0, 0, 0};
  if (p->d_tri_perm) {  // blocked output maps of the final pass (k_fin2)
    unsigned long long* fl = (unsigned long long*)stats.p + 2;
    k_blocked_check<<<grid_1d(A), 256, 0, st>>>(p->d_tri_inv_elem, A, A >> 4, fl);
    k_blocked_check<<<grid_1d(A), 256, 0, st>>>(p->d_tri_inv_node, A, A >> 4, fl + 1);
  }
  if (p->d_tri_perm && cudaMemcpyAsync(p->tri_front_tw, p->d_twiddles, csz * std::min<int64_t>(31, A - 1),
                                       cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "plan build"));
  if (cudaGetLastError() != cudaSuccess ||
      cudaMemcpyAsync(h, stats.p, 32, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return done(cuda_fail(cudaGetLastError(), "plan build"));
  p->n_nodes = (int64_t)h[0];
  p->mu_star = (int64_t)h[1];
  p->tri_blocked_elem = p->d_tri_perm && h[2] != 0;
  p->tri_blocked_node = p->d_tri_perm && h[3] != 0;
  trace.mark("stats readback");
  static const bool cf = [] {
    const char* e = getenv("SFFT_TRI_CF");
    return !(e && atoi(e) == 0);
  }();
  // head-path plans: the conflict-free epilogue tables are opt-in
  // (SFFT_HEAD_CF=1: k_head 46.1 -> 43.3 us per chunk, the step unchanged at
  // 126.5-126.9 us, and the host Euler splits add ~4 ms to the plan build)
  static const bool head_cf = [] {
    const char* e = getenv("SFFT_HEAD_CF");
    return e && atoi(e) == 1;
  }();
  if (p->d_tri_perm && dtype == SFFT_C64 && cf) {
    if ((rc = head_covers(p) ? (head_cf ? head_conflict_free_tables(p, st) : SFFT_OK)
                             : tri_conflict_free_tables(p, st)))
      return done(rc);
  }
  trace.mark("conflict-free tables");
  *out_plan = p;
  return SFFT_OK;
}

// ------------------------------------------------------ congruence tree ---
//
// T^depth(J) (congruence.py:134-222): level l holds one node per residue
// class mod 2^l that meets J, in ascending residue order, its members in
// ascending j.  Sorting J by K_l = rotr_M(j, l) = (j mod 2^l) 2^(M-l) +
// (j >> l) gives exactly that order (the key is a bijection of j, so the
// bit-map rank sorts it); a node starts where two neighbours differ in the
// low l bits.  One rank per level, O(k + 2^M / 32) work each.
__global__ void k_tree_keys(const int64_t* __restrict__ J, int64_t k, int M, int l, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ bitmap) {
  const uint32_t lowmask = l >= 32 ? 0xffffffffu : ((1u << l) - 1u);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)J[e];
    const uint32_t key = l == 0 ? j : (((j & lowmask) << (M - l)) | (j >> l));
    keys[e] = key;
    atomicOr(&bitmap[key >> 5], 1u << (key & 31));
  }
}
__global__ void k_tree_scatter(const int64_t* __restrict__ J, const uint32_t* __restrict__ keys, int64_t k,
                               const uint32_t* __restrict__ bitmap, const uint32_t* __restrict__ wprefix,
                               const uint32_t* __restrict__ bprefix, int64_t* __restrict__ members) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x)
    members[bit_rank(keys[e], bitmap, wprefix, bprefix)] = J[e];
}
// node starts: a k-bit bitmap of positions where the residue mod 2^l changes
__global__ void k_tree_starts(const int64_t* __restrict__ members, int64_t k, int l, uint32_t* __restrict__ sbits) {
  const int64_t lowmask = (1ll << l) - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x)
    if (p == 0 || ((members[p] ^ members[p - 1]) & lowmask) != 0) atomicOr(&sbits[p >> 5], 1u << (p & 31));
}
__global__ void k_tree_offsets(const uint32_t* __restrict__ sbits, int64_t k, const uint32_t* __restrict__ wprefix,
                               const uint32_t* __restrict__ bprefix, int32_t* __restrict__ node_off,
                               int32_t* __restrict__ n_nodes) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < k; p += (int64_t)gridDim.x * blockDim.x) {
    if (!((sbits[p >> 5] >> (p & 31)) & 1u)) continue;
    const uint32_t r = bit_rank((uint32_t)p, sbits, wprefix, bprefix);
    node_off[r] = (int32_t)p;
    if (p == 0) {
      // total node count = rank of k (one past the last bit), written by thread 0
      const int64_t last = k - 1;
      uint32_t cnt = bit_rank((uint32_t)last, sbits, wprefix, bprefix) + ((sbits[last >> 5] >> (last & 31)) & 1u);
      *n_nodes = (int32_t)cnt;
    }
  }
}
__global__ void k_tree_close(int32_t* __restrict__ node_off, const int32_t* __restrict__ n_nodes, int64_t k) {
  node_off[*n_nodes] = (int32_t)k;
}

extern "C" int sfft_tree_build(const int64_t* J, int64_t k, int M, int level_lo, int level_hi, int64_t* members,
                               int32_t* node_off, int32_t* n_nodes, sfft_stream_t stream) {
  SFFT_NVTX("sfft_tree_build");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 28) return fail(SFFT_ERR_UNSUPPORTED, "congruence tree on the device needs 1 <= M <= 28");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (level_lo < 0 || level_hi < level_lo || level_hi > M)
    return fail(SFFT_ERR_INVALID, "depth must be in [0, " + std::to_string(M) + "]");
  if (!members || !node_off || !n_nodes) return fail(SFFT_ERR_INVALID, "null output");
  DevBuf tmpJ;
  const int64_t* dJ = nullptr;
  int rc;
  if ((rc = to_device_J(J, k, st, tmpJ, &dJ))) return rc;
  uint64_t mask = 0;
  if ((rc = analyze_device(dJ, k, M, &mask, st))) return rc;  // validates J (sorted, distinct, in range)
  const int nl = level_hi - level_lo + 1;
  DevBuf keys, dm, doff, dn;
  if ((rc = alloc(keys, 4 * k, st))) return rc;
  const bool dev_out = is_device_pointer(members) && is_device_pointer(node_off) && is_device_pointer(n_nodes);
  int64_t* m_out = members;
  int32_t* o_out = node_off;
  int32_t* n_out = n_nodes;
  if (!dev_out) {
    if ((rc = alloc(dm, 8 * k * (size_t)nl, st))) return rc;
    if ((rc = alloc(doff, 4 * (k + 1) * (size_t)nl, st))) return rc;
    if ((rc = alloc(dn, 4 * (size_t)nl, st))) return rc;
    m_out = (int64_t*)dm.p;
    o_out = (int32_t*)doff.p;
    n_out = (int32_t*)dn.p;
  }
  for (int l = level_lo; l <= level_hi; ++l) {
    const int i = l - level_lo;
    int64_t* mem = m_out + (size_t)i * k;
    int32_t* off = o_out + (size_t)i * (k + 1);
    {
      RankCtx R;
      if ((rc = rank_prepare(R, nullptr, nullptr, k, M, st))) return rc;
      k_tree_keys<<<grid_1d(k), 256, 0, st>>>(dJ, k, M, l, (uint32_t*)keys.p, (uint32_t*)R.bitmap.p);
      if ((rc = rank_scan(R, st))) return rc;
      k_tree_scatter<<<grid_1d(k), 256, 0, st>>>(dJ, (const uint32_t*)keys.p, k, (const uint32_t*)R.bitmap.p,
                                                 (const uint32_t*)R.wprefix.p, (const uint32_t*)R.bsum.p, mem);
    }
    {
      RankCtx R;
      int lg = 0;
      while ((1ll << lg) < k) ++lg;
      if ((rc = rank_prepare(R, nullptr, nullptr, k, std::max(lg, 5), st))) return rc;
      k_tree_starts<<<grid_1d(k), 256, 0, st>>>(mem, k, l, (uint32_t*)R.bitmap.p);
      if ((rc = rank_scan(R, st))) return rc;
      k_tree_offsets<<<grid_1d(k), 256, 0, st>>>((const uint32_t*)R.bitmap.p, k, (const uint32_t*)R.wprefix.p,
                                                 (const uint32_t*)R.bsum.p, off, n_out + i);
      k_tree_close<<<1, 1, 0, st>>>(off, n_out + i, k);
    }
  }
  SFFT_CUDA(cudaGetLastError());
  if (!dev_out) {  // host (or mixed host / device) outputs: copied back, synchronous
    SFFT_CUDA(cudaMemcpyAsync(members, m_out, 8 * k * (size_t)nl, cudaMemcpyDefault, st));
    SFFT_CUDA(cudaMemcpyAsync(node_off, o_out, 4 * (k + 1) * (size_t)nl, cudaMemcpyDefault, st));
    SFFT_CUDA(cudaMemcpyAsync(n_nodes, n_out, 4 * (size_t)nl, cudaMemcpyDefault, st));
    SFFT_CUDA(cudaStreamSynchronize(st));
  }
  return SFFT_OK;
}

extern "C" int sfft_plan_batched(const int64_t* J, int64_t k, int64_t n_supports, int M, int dtype,
                                 sfft_stream_t stream, sfft_plan** out_plan) {
  SFFT_NVTX("sfft_plan_batched");
  cudaStream_t st = (cudaStream_t)stream;
  if (!out_plan) return fail(SFFT_ERR_INVALID, "null plan output");
  *out_plan = nullptr;
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (dtype != SFFT_C64 && dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown dtype");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (n_supports < 1) return fail(SFFT_ERR_INVALID, "n_supports must be >= 1");
  if (!J) return fail(SFFT_ERR_INVALID, "null support pointer");
  if (k & (k - 1)) return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support");
  sfft_plan* p = new sfft_plan();
  std::memset(p, 0, sizeof(*p));
  SFFT_CUDA(cudaGetDevice(&p->device));
  p->per_signal = 1;
  p->n_supports = n_supports;
  p->M = M;
  p->dtype = dtype;
  p->k = k;
  p->A = k;
  p->s = 63 - __builtin_clzll((unsigned long long)k);
  p->n_r = p->s;
  p->n_nodes = k;
  p->mu_star = 1;
  p->homogeneous = 1;
  const size_t bytes = sizeof(int64_t) * (size_t)k * (size_t)n_supports;
  cudaError_t e = cudaMalloc((void**)&p->d_J, bytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->d_J, J, bytes, cudaMemcpyDefault, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    plan_free(p);
    return cuda_fail(e, "per-signal plan");
  }
  *out_plan = p;
  return SFFT_OK;
}

extern "C" int sfft_plan_destroy(sfft_plan* plan) {
  plan_free(plan);
  return SFFT_OK;
}

extern "C" int sfft_plan_get_info(const sfft_plan* p, sfft_plan_info* info) {
  if (!p || !info) return fail(SFFT_ERR_INVALID, "null plan or info");
  std::memset(info, 0, sizeof(*info));
  info->M = p->M;
  info->dtype = p->dtype;
  info->n_r = p->n_r;
  info->height = p->height;
  info->s = p->s;
  info->level = p->level;
  info->homogeneous = p->homogeneous;
  info->k = p->k;
  info->A = p->A;
  info->n_nodes = p->n_nodes;
  info->mu_star = p->mu_star;
  info->pivot_mask = p->pivot_mask;
  info->per_signal = p->per_signal;
  for (int i = 0; i < 32; ++i) info->used[i] = i < p->s ? p->used[i] : 0;
  return SFFT_OK;
}

static int copy_out(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  SFFT_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  return SFFT_OK;
}

extern "C" int sfft_plan_tables(const sfft_plan* p, int64_t* element_slots, int64_t* slot_residues,
                                uint8_t* slot_real, int64_t* node_residues, int64_t* offsets, void* twiddles,
                                sfft_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!p) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(p, "sfft_plan_tables")) return rj;
  int rc;
  DevBuf w, du;
  const int64_t big = std::max(std::max(p->k, p->A), p->n_nodes);
  if ((rc = alloc(w, 8 * big, st))) return rc;
  int64_t* dw = (int64_t*)w.p;
  auto widen = [&](const int32_t* src, int64_t n, int64_t* dst) -> int {
    if (!dst) return SFFT_OK;
    k_widen<<<grid_1d(n), 256, 0, st>>>(src, n, dw);
    return copy_out(dst, dw, 8 * n, st) ? SFFT_ERR_CUDA : (cudaStreamSynchronize(st) == cudaSuccess ? SFFT_OK : SFFT_ERR_CUDA);
  };
  if ((rc = widen(p->d_element_slots, p->k, element_slots))) return rc;
  if ((rc = widen(p->d_slot_residues, p->A, slot_residues))) return rc;
  if ((rc = widen(p->d_node_residues, p->n_nodes, node_residues))) return rc;
  if (slot_real && (rc = copy_out(slot_real, p->d_slot_real, p->A, st))) return rc;
  if (twiddles && p->A > 1 &&
      (rc = copy_out(twiddles, p->d_twiddles, (p->dtype == SFFT_C64 ? 8 : 16) * (p->A - 1), st)))
    return rc;
  if (offsets) {
    if ((rc = alloc(du, 4 * 32, st))) return rc;
    SFFT_CUDA(cudaMemcpyAsync(du.p, p->used, 4 * 32, cudaMemcpyHostToDevice, st));
    k_offsets<<<grid_1d(p->A), 256, 0, st>>>((const int32_t*)du.p, p->s, p->M, p->A, dw, 0);
    if ((rc = copy_out(offsets, dw, 8 * p->A, st))) return rc;
  }
  SFFT_CUDA(cudaStreamSynchronize(st));
  return SFFT_OK;
}

// ------------------------------------------------ SAS prefix weight profile ---
// For the prefixes p[:t] (t = 0..s) of the pivot list of J, the congruence-tree
// nodes at level p[t-1]+1 are the classes of the first t pattern bits (J has
// no other pivot below p[t-1]), so one pass over J fills all prefix
// histograms; mu*(t) = max weight, sum w^2 (sas.py:80-86, 105-113).
__global__ void k_prefix_hist(const int64_t* __restrict__ J, int64_t k, const int32_t* __restrict__ piv, int s,
                              uint32_t* __restrict__ hist) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t j = (uint64_t)J[e];
    uint32_t pat = 0;
    atomicAdd(&hist[0], 1u);  // t = 0: the root
    for (int t = 1; t <= s; ++t) {
      pat |= (uint32_t)((j >> piv[t - 1]) & 1u) << (t - 1);
      atomicAdd(&hist[((1u << t) - 1) + pat], 1u);
    }
  }
}

__global__ void k_prefix_reduce(const uint32_t* __restrict__ hist, int s, unsigned long long* __restrict__ out) {
  // out[2t] = max weight, out[2t+1] = sum of squared weights, for t = 0..s
  for (int t = blockIdx.x; t <= s; t += gridDim.x) {
    const uint32_t* h = hist + ((1u << t) - 1);
    unsigned long long mx = 0, sq = 0;
    for (int64_t i = threadIdx.x; i < (1ll << t); i += blockDim.x) {
      const unsigned long long w = h[i];
      mx = mx > w ? mx : w;
      sq += w * w;
    }
    for (int d = 16; d > 0; d >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, d);
      mx = mx > o ? mx : o;
      sq += __shfl_xor_sync(0xffffffffu, sq, d);
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&out[2 * t], mx);
      atomicAdd(&out[2 * t + 1], sq);
    }
  }
}

extern "C" int sfft_prefix_weights(const int64_t* J, int64_t k, int M, const int32_t* piv, int s,
                                   uint64_t* mu_out, uint64_t* sumsq_out, sfft_stream_t stream) {
  SFFT_NVTX("sfft_prefix_weights");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (s < 0 || s > 26) return fail(SFFT_ERR_UNSUPPORTED, "prefix profile limited to 26 pivots");
  int rc;
  DevBuf tmpJ, dpiv, hist, out;
  const int64_t* dJ = nullptr;
  if ((rc = to_device_J(J, k, st, tmpJ, &dJ))) return rc;
  if ((rc = alloc(dpiv, 4 * std::max(s, 1), st))) return rc;
  if ((rc = alloc(hist, 4 * ((2ll << s) - 1), st))) return rc;
  if ((rc = alloc(out, 16 * (s + 1), st))) return rc;
  if (s) SFFT_CUDA(cudaMemcpyAsync(dpiv.p, piv, 4 * s, cudaMemcpyHostToDevice, st));
  SFFT_CUDA(cudaMemsetAsync(hist.p, 0, 4 * ((2ll << s) - 1), st));
  SFFT_CUDA(cudaMemsetAsync(out.p, 0, 16 * (s + 1), st));
  k_prefix_hist<<<grid_1d(k), 256, 0, st>>>(dJ, k, (const int32_t*)dpiv.p, s, (uint32_t*)hist.p);
  k_prefix_reduce<<<s + 1, 256, 0, st>>>((const uint32_t*)hist.p, s, (unsigned long long*)out.p);
  SFFT_CUDA(cudaGetLastError());
  std::vector<unsigned long long> h(2 * (s + 1));
  SFFT_CUDA(cudaMemcpyAsync(h.data(), out.p, 16 * (s + 1), cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  for (int t = 0; t <= s; ++t) {
    mu_out[t] = h[2 * t];
    sumsq_out[t] = h[2 * t + 1];
  }
  return SFFT_OK;
}
