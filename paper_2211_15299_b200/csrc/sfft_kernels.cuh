// Device building blocks shared by the transform kernels (sfft_hidft.cu,
// sfft_split.cu, sfft_fused.cu): slot geometry, the swizzled shared-memory
// layout, the register-blocked butterfly, the pass-0 gather, the launch
// arguments of the plan-driven kernels and the occupancy cache.
#pragma once

#include <map>
#include <mutex>
#include <utility>

#include "sfft_common.cuh"
#include "sfft_plan.h"

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
template <typename T, int S, typename In = T, int EOV = 0>
__device__ __forceinline__ void gather(Cx<T> (&v)[Geo<T, S, EOV>::E], int t, const Cx<In>* __restrict__ row,
                                       const uint32_t (&d)[S > 0 ? S : 1], uint32_t base, uint32_t nmask) {
  using G = Geo<T, S, EOV>;
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

// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; griddepcontrol.wait blocks until the predecessor has
// completed and its writes are visible (a no-op without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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
  int debug_skip;  // split-pass ablation probes only (SFFT_SPLIT_DEBUG, tools/split_time.py)
};

template <typename T, int S> constexpr size_t plan_smem() {
  return (size_t)Geo<T, S>::SPC * Geo<T, S>::A * sizeof(Cx<T>);
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Per (kernel, device): opt in to the full dynamic shared memory and cache
// the occupancy (resident CTAs per SM).
inline std::mutex g_kmu;
inline std::map<std::pair<const void*, int>, int> g_occ;

template <typename K>
inline int kernel_occupancy(K kernel, int nt, size_t smem, int* occ) {
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
  int smem_max = 0;
  SFFT_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (smem > (size_t)smem_max)
    return fail(SFFT_ERR_UNSUPPORTED, "kernel needs " + std::to_string(smem) + " B of shared memory, the device " +
                                          "allows " + std::to_string(smem_max));
  SFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int o = 0;
  SFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, nt, smem));
  if (o < 1) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    return fail(SFFT_ERR_UNSUPPORTED, "kernel does not fit on an SM (" + std::to_string(nt) + " threads x " +
                                          std::to_string(fa.numRegs) + " registers, " + std::to_string(smem) +
                                          " B dynamic + " + std::to_string(fa.sharedSizeBytes) +
                                          " B static shared memory, max threads " +
                                          std::to_string(fa.maxThreadsPerBlock) + ")");
  }
  std::lock_guard<std::mutex> lk(g_kmu);
  g_occ[key] = o;
  *occ = o;
  return SFFT_OK;
}

// 2^s beyond one CTA (sfft_split.cu): the two-pass split transform and the
// number of launches it issues for `rows` rows
int run_large(const sfft_plan* p, const PlanArgs& a, const int32_t* inv1, cudaStream_t st);
int large_launch_count(const sfft_plan* p, int64_t rows, int64_t* launches);

}  // namespace sfft
