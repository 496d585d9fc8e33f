// Shared device/host helpers for the B200 Hi-DFT library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "structfft_b200.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no cost without an attached tool

namespace sfft {

// NVTX range over one C-ABI call (nsys / ncu --nvtx show the library's calls
// as named ranges around their kernels); SFFT_NVTX(name) at function entry
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define SFFT_NVTX(name) ::sfft::NvtxRange sfft_nvtx_range__(name)

// ------------------------------------------------------------ complex ---
template <typename T> struct Cx;
template <> struct __align__(8) Cx<float> { float x, y; };
template <> struct __align__(16) Cx<double> { double x, y; };

template <typename T>
__device__ __forceinline__ Cx<T> cadd(Cx<T> a, Cx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T>
__device__ __forceinline__ Cx<T> csub(Cx<T> a, Cx<T> b) { return {a.x - b.x, a.y - b.y}; }
template <typename T>
__device__ __forceinline__ Cx<T> cmul(Cx<T> a, Cx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ Cx<T> cscale(Cx<T> a, T s) { return {a.x * s, a.y * s}; }

// Generalised radix-2 butterfly (hidft.py:163-164): branch 0 = u - w v,
// branch 1 = u + w v.  Computed as p = u + w v (4 FMAs) and u - w v = 2u - p
// (2 FMAs): 6 FP instructions instead of 8, same error order (one rounding
// of |u| + |w v| magnitude per output component).
__device__ __forceinline__ void bfly(Cx<float>& u, Cx<float>& v, Cx<float> w) {
  const float px = fmaf(w.x, v.x, fmaf(-w.y, v.y, u.x));
  const float py = fmaf(w.x, v.y, fmaf(w.y, v.x, u.y));
  u = {fmaf(2.f, u.x, -px), fmaf(2.f, u.y, -py)};
  v = {px, py};
}
__device__ __forceinline__ void bfly(Cx<double>& u, Cx<double>& v, Cx<double> w) {
  const double px = fma(w.x, v.x, fma(-w.y, v.y, u.x));
  const double py = fma(w.x, v.y, fma(w.y, v.x, u.y));
  u = {fma(2.0, u.x, -px), fma(2.0, u.y, -py)};
  v = {px, py};
}

// Packed-fp32 butterfly (sm_100 FFMA2: two fp32 FMAs per instruction).  With
// w v = v.x w + v.y (i w), i w = (-w.y, w.x):  p = u + v.x w + v.y iw,
// u' = 2u - p: three FFMA2 instead of six FFMA (same roundings as bfly).
// iw is passed in so that a twiddle shared by several butterflies is
// rotated once.
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ Cx<float> upk2(unsigned long long r) {
  Cx<float> v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ Cx<float> rot_i(Cx<float> w) { return {-w.y, w.x}; }
__device__ __forceinline__ void bfly2(Cx<float>& u, Cx<float>& v, Cx<float> w, Cx<float> iw) {
  const unsigned long long U = pk2(u.x, u.y);
  unsigned long long P = ffma2(pk2(v.x, v.x), pk2(w.x, w.y), U);
  P = ffma2(pk2(v.y, v.y), pk2(iw.x, iw.y), P);
  const Cx<float> p = upk2(P);
  u = upk2(ffma2(pk2(2.f, 2.f), U, pk2(-p.x, -p.y)));
  v = p;
}

// Streaming sample loads: one sector per sample in the sparse patterns, no
// reuse through L1, so bypass L1 allocation.
__device__ __forceinline__ Cx<float> load_sample(const Cx<float>* p) {
  Cx<float> r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
               : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ Cx<double> load_sample(const Cx<double>* p) {
  Cx<double> r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

// Twiddle exp(-2 pi i (shared + 2^rk) / 2^(rk+1)) (hidft.py:83), evaluated
// with an exact reduced argument: u = (shared + 2^rk) mod 2^(rk+1), angle
// -u/2^rk in units of pi.
__device__ __forceinline__ void twiddle_d(uint32_t shared, int rk, double& c, double& s) {
  const uint64_t u = ((uint64_t)shared + (1ull << rk)) & ((2ull << rk) - 1);
  const double th = -(double)u * ldexp(1.0, -rk);
  sincospi(th, &s, &c);
}
template <typename T> __device__ __forceinline__ Cx<T> twiddle(uint32_t shared, int rk);
template <> __device__ __forceinline__ Cx<double> twiddle<double>(uint32_t shared, int rk) {
  double c, s;
  twiddle_d(shared, rk, c, s);
  return {c, s};
}
template <> __device__ __forceinline__ Cx<float> twiddle<float>(uint32_t shared, int rk) {
  if (rk < 23) {  // u < 2^24: the fp32 argument is exact, sincospif is ~1 ulp
    const uint32_t u = (shared + (1u << rk)) & ((2u << rk) - 1);
    const float th = -(float)u * ldexpf(1.0f, -rk);
    float s, c;
    sincospif(th, &s, &c);
    return {c, s};
  }
  double c, s;
  twiddle_d(shared, rk, c, s);
  return {(float)c, (float)s};
}

// bit extract: pattern bits of j at the pivot positions piv[0..s)
__device__ __forceinline__ uint32_t pext_pivots(uint32_t j, const int* piv, int s) {
  uint32_t p = 0;
  for (int i = 0; i < s; ++i) p |= ((j >> piv[i]) & 1u) << i;
  return p;
}

// ------------------------------------------------------------ host side ---
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define SFFT_CUDA(call)                                        \
  do {                                                         \
    cudaError_t e__ = (call);                                  \
    if (e__ != cudaSuccess) return ::sfft::cuda_fail(e__, #call); \
  } while (0)

bool is_device_pointer(const void* p);
int num_sms();

}  // namespace sfft
