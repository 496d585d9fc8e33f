// Shift-and-sample decoding on the device for mu* > 1 (reference sas.py).
//
//   (N/|I|) * Hidft(tau^j f)(v) = sum_{l in v} Ff(l) x_l^j,  x_l = e^{-2 pi i l/N}
//
// for j < m_v (the node's weight), one Vandermonde system per aliased node v
// at the decode level (sas.py:1-12).  The mu* shifted Hi-DFTs run as one
// launch of the transform kernels (B*mu* rows).  This file decodes:
//   * Bjorck-Pereyra with Leja ordering in float64 (sas.py:135-203), the
//     reference's forward-error estimate (sas.py:214-235);
//   * nodes estimated above tolerance/20 are re-measured and re-solved in
//     double-double (sas.py:290-310, _ddc.py), with double-double roots
//     computed on the device (Taylor series after exact reduction) in the
//     reference's coarse x fine table layout (_ddc.py:151-205);
//   * non-escalated nodes whose residual exceeds max(tol, 1e-9) fall back to
//     a dense LU solve with partial pivoting (sas.py:386-395).

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "sfft_common.cuh"
#include "sfft_plan.h"

namespace sfft {

constexpr int kMaxMu = 64;       // node weights decoded one (signal, node) per thread, arrays in registers
constexpr int kMaxMuBig = 1024;  // heavier nodes: one CTA per (signal, node), arrays in shared memory

// ------------------------------------------------------ double-double ---
// Same formulas as _ddc.py (no FMA contraction: explicit _rn intrinsics);
// two_prod uses the exact FMA error term (equal to Dekker's split result).
struct dd {
  double hi, lo;
};
struct cdd {
  dd re, im;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double err = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, err};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  const dd s = two_sum(x.hi, y.hi);
  const double e = __dadd_rn(__dadd_rn(s.lo, x.lo), y.lo);
  return quick_two_sum(s.hi, e);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }
__device__ __forceinline__ dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
__device__ __forceinline__ dd dd_mul(dd x, dd y) {
  const dd p = two_prod(x.hi, y.hi);
  const double e = __dadd_rn(__dadd_rn(p.lo, __dmul_rn(x.hi, y.lo)), __dmul_rn(x.lo, y.hi));
  return quick_two_sum(p.hi, e);
}
__device__ __forceinline__ dd dd_mul_f(dd x, double f) {
  const dd p = two_prod(x.hi, f);
  return quick_two_sum(p.hi, __dadd_rn(p.lo, __dmul_rn(x.lo, f)));
}
__device__ __forceinline__ dd dd_div(dd x, dd y) {
  const double q1 = __ddiv_rn(x.hi, y.hi);
  dd r = dd_sub(x, dd_mul_f(y, q1));
  const double q2 = __ddiv_rn(r.hi, y.hi);
  r = dd_sub(r, dd_mul_f(y, q2));
  const double q3 = __ddiv_rn(r.hi, y.hi);
  return dd_add(quick_two_sum(q1, q2), dd{q3, 0.0});
}
__device__ __forceinline__ cdd cdd_add(cdd u, cdd v) { return {dd_add(u.re, v.re), dd_add(u.im, v.im)}; }
__device__ __forceinline__ cdd cdd_sub(cdd u, cdd v) { return {dd_sub(u.re, v.re), dd_sub(u.im, v.im)}; }
__device__ __forceinline__ cdd cdd_mul(cdd u, cdd v) {
  return {dd_sub(dd_mul(u.re, v.re), dd_mul(u.im, v.im)), dd_add(dd_mul(u.re, v.im), dd_mul(u.im, v.re))};
}
__device__ __forceinline__ cdd cdd_mul_complex(cdd u, double a, double b) {
  return {dd_sub(dd_mul_f(u.re, a), dd_mul_f(u.im, b)), dd_add(dd_mul_f(u.re, b), dd_mul_f(u.im, a))};
}
__device__ __forceinline__ cdd cdd_div(cdd u, cdd v) {
  const dd den = dd_add(dd_mul(v.re, v.re), dd_mul(v.im, v.im));
  const dd re = dd_add(dd_mul(u.re, v.re), dd_mul(u.im, v.im));
  const dd im = dd_sub(dd_mul(u.im, v.re), dd_mul(u.re, v.im));
  return {dd_div(re, den), dd_div(im, den)};
}

// e^{+2 pi i t / D} in double-double, D a power of two, 0 <= t < D.
// Exact reduction: 4t/D = q + r exactly; angle = q*pi/2 + r*pi/2, reflected
// to phi = (pi/2) * min(r, 1-r) in [0, pi/4]; Taylor series to 1e-33.
__device__ cdd dd_root(uint64_t t, int logD) {
  const dd PIO2 = {1.5707963267948966, 6.123233995736766e-17};
  const double v4 = ldexp((double)t, 2 - logD);  // 4t/D, exact
  const int q = (int)floor(v4);
  double r = v4 - (double)q;
  const bool refl = r > 0.5;
  if (refl) r = 1.0 - r;
  const dd phi = dd_mul_f(PIO2, r);
  const dd x2 = dd_mul(phi, phi);
  dd s = phi, c = {1.0, 0.0}, ts = phi, tc = {1.0, 0.0};
  for (int n = 1; n <= 15; ++n) {
    ts = dd_div(dd_mul(ts, x2), dd{(double)((2 * n) * (2 * n + 1)), 0.0});
    tc = dd_div(dd_mul(tc, x2), dd{(double)((2 * n - 1) * (2 * n)), 0.0});
    if (n & 1) {
      s = dd_sub(s, ts);
      c = dd_sub(c, tc);
    } else {
      s = dd_add(s, ts);
      c = dd_add(c, tc);
    }
  }
  dd cs = refl ? s : c, sn = refl ? c : s;  // cos/sin of (pi/2) r
  switch (q & 3) {
    case 0: return {cs, sn};
    case 1: return {dd_neg(sn), cs};
    case 2: return {dd_neg(cs), dd_neg(sn)};
    default: return {sn, dd_neg(cs)};
  }
}

// root table of _ddc.py:151-205: fine[s] = e^{2 pi i s / N}, s < 2^h;
// coarse[q] = e^{2 pi i q / 2^(M-h)}; root(t) = coarse[t >> h] * fine[t & (2^h-1)]
__global__ void k_root_tables(cdd* __restrict__ fine, cdd* __restrict__ coarse, int M) {
  const int h = M / 2;
  const int64_t nf = 1ll << h, nc = 1ll << (M - h);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf + nc; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nf) fine[i] = dd_root((uint64_t)i, M);
    else coarse[i - nf] = dd_root((uint64_t)(i - nf), M - h);
  }
}

struct RootTab {
  const cdd* fine;
  const cdd* coarse;
  int h;
  uint64_t nmask;
  __device__ __forceinline__ cdd get(uint64_t t) const {
    t &= nmask;
    return cdd_mul(coarse[t >> h], fine[t & ((1ull << h) - 1)]);
  }
};

// ------------------------------------------------ float64 node decoding ---
struct C64x {  // complex double with plain arithmetic (reference numpy complex128)
  double x, y;
};
__device__ __forceinline__ C64x cm(C64x a, C64x b) { return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ C64x cs(C64x a, C64x b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ C64x cdv(C64x a, C64x b) {
  // numpy complex division (Smith's algorithm)
  if (fabs(b.x) >= fabs(b.y)) {
    const double rat = b.y / b.x, scl = 1.0 / (b.x + b.y * rat);
    return {(a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl};
  }
  const double rat = b.x / b.y, scl = 1.0 / (b.y + b.x * rat);
  return {(a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl};
}
__device__ __forceinline__ double cabs2(C64x a) { return hypot(a.x, a.y); }

// sas.py:153-163 on nodes x[perm]
__device__ void bp_core(const C64x* x, const int* perm, C64x* c, int n) {
  for (int k = 0; k < n - 1; ++k)
    for (int j = n - 1; j > k; --j) c[j] = cs(c[j], cm(x[perm[k]], c[j - 1]));
  for (int k = n - 2; k >= 0; --k) {
    for (int j = k + 1; j < n; ++j) c[j] = cdv(c[j], cs(x[perm[j]], x[perm[j - k - 1]]));
    for (int j = k; j < n - 1; ++j) c[j] = cs(c[j], c[j + 1]);
  }
}

// sas.py:135-150 (scratch: prod, chosen of n entries)
__device__ void leja_order_s(const C64x* x, int n, int* order, double* prod, bool* chosen) {
  int i0 = 0;
  double best = -1.0;
  for (int i = 0; i < n; ++i) {
    const double a = cabs2(x[i]);
    if (a > best) { best = a; i0 = i; }
    chosen[i] = false;
  }
  order[0] = i0;
  chosen[i0] = true;
  for (int i = 0; i < n; ++i) prod[i] = cabs2(cs(x[i], x[i0]));
  for (int t = 1; t < n; ++t) {
    int ib = 0;
    double pb = -2.0;
    for (int i = 0; i < n; ++i) {
      const double pm = chosen[i] ? -1.0 : prod[i];
      if (pm > pb) { pb = pm; ib = i; }
    }
    order[t] = ib;
    chosen[ib] = true;
    for (int i = 0; i < n; ++i) prod[i] *= cabs2(cs(x[i], x[ib]));
  }
}
__device__ void leja_order(const C64x* x, int n, int* order) {
  double prod[kMaxMu];
  bool chosen[kMaxMu];
  leja_order_s(x, n, order, prod, chosen);
}

// vandermonde_solve (sas.py:166-203): c[perm] = bp_core(x[perm], y)
__device__ void vandermonde_solve_s(const C64x* x, const C64x* y, int n, const int* perm, C64x* out, C64x* c) {
  for (int i = 0; i < n; ++i) c[i] = y[i];
  bp_core(x, perm, c, n);
  for (int i = 0; i < n; ++i) out[perm[i]] = c[i];
}
__device__ void vandermonde_solve(const C64x* x, const C64x* y, int n, const int* perm, C64x* out) {
  C64x c[kMaxMu];
  vandermonde_solve_s(x, y, n, perm, out, c);
}

// out[j] = sum_m x_m^j c_m, the powers by repeated multiplication and each
// sum in increasing m (the same operations as forming V row by row), O(n^2)
__device__ void forward_apply(const C64x* x, const C64x* c, int n, C64x* out) {
  for (int j = 0; j < n; ++j) out[j] = {0.0, 0.0};
  for (int m = 0; m < n; ++m) {
    C64x p = {1.0, 0.0};
    for (int j = 0; j < n; ++j) {
      if (j) p = cm(p, x[m]);
      out[j] = {out[j].x + (p.x * c[m].x - p.y * c[m].y), out[j].y + (p.x * c[m].y + p.y * c[m].x)};
    }
  }
}

struct SasDecodeArgs {
  const void* nodevals;  // (B*mu) rows x n_nodes, row r = signal r/mu, shift r%mu
  int64_t ld_nv;
  int nv_c64;
  int64_t B, mu, n_nodes, k;
  int M;
  double scale, tol;
  const int32_t* node_off;  // n_nodes+1
  const int32_t* node_mem;  // k element indices
  const int64_t* J;         // k support indices
  void* out;                // B x k complex128
  int64_t ld_out;
  int32_t* flags;  // B x n_nodes: bit0 escalate, bit1 dense fallback
  double* resid;   // B x n_nodes residual (sas.py:386-388)
  const C64x* node_x;        // per-plan node tables (k_node_prep)
  const int32_t* node_perm;
  const double* node_amp;
  int32_t* esc_list;         // (signal, node) ids to escalate / to refactor densely,
  int32_t* fb_list;          // appended in any order (each node is decoded on its own)
  int32_t* big_list;         // (signal, node) ids of weight > kMaxMu (k_sas_decode_f64_big)
  unsigned int* counts;      // [3] lengths of esc_list / fb_list / big_list
};

__device__ __forceinline__ C64x nodeval(const SasDecodeArgs& a, int64_t row, int64_t node) {
  if (a.nv_c64) {
    const float2 v = reinterpret_cast<const float2*>(a.nodevals)[row * a.ld_nv + node];
    return {(double)v.x, (double)v.y};
  }
  const double2 v = reinterpret_cast<const double2*>(a.nodevals)[row * a.ld_nv + node];
  return {v.x, v.y};
}

// ||inv(V)||_inf in O(m^2): row q of inv(V) (V[j][m] = x_m^j) holds the
// coefficients of the Lagrange basis L_q(z) = P(z) / ((z - x_q) P'(x_q)),
// P(z) = prod_i (z - x_i); synthetic division per node (the reference
// inverts V densely, sas.py:229-233; this is the same norm)
__device__ double lagrange_inv_norm_s(const C64x* x, int m, C64x* P) {  // P: m + 1 entries
  double amp = 0.0;
  P[0] = {1.0, 0.0};
  for (int i = 1; i <= m; ++i) P[i] = {0.0, 0.0};
  for (int i = 0; i < m; ++i)  // multiply by (z - x_i)
    for (int e = i + 1; e >= 0; --e) P[e] = cs(e ? P[e - 1] : C64x{0.0, 0.0}, cm(x[i], P[e]));
  for (int q = 0; q < m; ++q) {
    C64x qc = P[m];  // Q(z) = P(z) / (z - x_q): leading coefficient
    C64x den = {1.0, 0.0};
    for (int i = 0; i < m; ++i)
      if (i != q) den = cm(den, cs(x[q], x[i]));
    const double dabs = cabs2(den);
    double row = cabs2(qc);
    for (int e = m - 1; e >= 1; --e) {
      const C64x t = cm(x[q], qc);
      qc = {P[e].x + t.x, P[e].y + t.y};
      row += cabs2(qc);
    }
    amp = fmax(amp, row / fmax(dabs, 1e-300));
  }
  return amp;
}
__device__ double lagrange_inv_norm(const C64x* x, int m) {
  C64x P[kMaxMu + 1];
  return lagrange_inv_norm_s(x, m, P);
}

// Per-node quantities that do not depend on the signal, computed once per
// plan: the nodes x_l = e^{-2 pi i l / N} of each member (node-member order),
// the Leja order (sas.py:135-150) and ||inv(V)||_inf (sas.py:229-233).
__global__ void k_node_prep(const int32_t* __restrict__ node_off, const int32_t* __restrict__ node_mem,
                            const int64_t* __restrict__ J, int64_t n_nodes, int M, C64x* __restrict__ node_x,
                            int32_t* __restrict__ node_perm, double* __restrict__ node_amp) {
  const double N = ldexp(1.0, M);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_nodes;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int off = node_off[v], m = node_off[v + 1] - off;
    if (m > kMaxMu) continue;  // k_node_prep_big
    C64x x[kMaxMu];
    int perm[kMaxMu];
    for (int j = 0; j < m; ++j) {
      const double l = (double)J[node_mem[off + j]];
      double sn, co;
      sincospi(-2.0 * l / N, &sn, &co);
      x[j] = {co, sn};
      node_x[off + j] = x[j];
    }
    if (m >= 3) {
      leja_order(x, m, perm);
    } else {
      for (int i = 0; i < m; ++i) perm[i] = i;
    }
    for (int j = 0; j < m; ++j) node_perm[off + j] = perm[j];
    node_amp[v] = m >= 2 ? lagrange_inv_norm(x, m) : 0.0;
  }
}

// k_node_prep for nodes heavier than kMaxMu: one CTA per node, its arrays in
// shared memory, the same sequential operations on thread 0
__global__ void k_node_prep_big(const int32_t* __restrict__ node_off, const int32_t* __restrict__ node_mem,
                                const int64_t* __restrict__ J, int64_t n_nodes, int M, C64x* __restrict__ node_x,
                                int32_t* __restrict__ node_perm, double* __restrict__ node_amp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const double N = ldexp(1.0, M);
  for (int64_t v = blockIdx.x; v < n_nodes; v += gridDim.x) {
    const int off = node_off[v], m = node_off[v + 1] - off;
    if (m <= kMaxMu || threadIdx.x != 0) continue;
    C64x* x = reinterpret_cast<C64x*>(smem_raw);  // m
    C64x* P = x + m;                                // m + 1
    double* prod = reinterpret_cast<double*>(P + m + 1);
    int* perm = reinterpret_cast<int*>(prod + m);
    bool* chosen = reinterpret_cast<bool*>(perm + m);
    for (int j = 0; j < m; ++j) {
      const double l = (double)J[node_mem[off + j]];
      double sn, co;
      sincospi(-2.0 * l / N, &sn, &co);
      x[j] = {co, sn};
      node_x[off + j] = x[j];
    }
    leja_order_s(x, m, perm, prod, chosen);
    for (int j = 0; j < m; ++j) node_perm[off + j] = perm[j];
    node_amp[v] = lagrange_inv_norm_s(x, m, P);
  }
}

// decode one (signal b, node v) of weight m (sas.py:343-399, float64 part):
// BP solve, forward-error estimate, residual; arrays are caller scratch
// (registers for m <= kMaxMu, shared memory above)
__device__ void decode_node(const SasDecodeArgs& a, int64_t b, int64_t v, int off, int m, C64x* x, C64x* y, C64x* c,
                            C64x* r, C64x* d, C64x* cs_scratch, int* perm) {
  const double noise_eps = 100.0 * 2.220446049250313e-16;
  const int64_t fid = b * a.n_nodes + v;  // flags / resid stay (signal, node) row-major
  C64x* out = reinterpret_cast<C64x*>(a.out) + b * a.ld_out;
  for (int j = 0; j < m; ++j) {
    const C64x raw = nodeval(a, b * a.mu + j, v);
    y[j] = {raw.x * a.scale, raw.y * a.scale};
    x[j] = a.node_x[off + j];  // per-plan tables (k_node_prep)
    perm[j] = a.node_perm[off + j];
  }
  vandermonde_solve_s(x, y, m, perm, c, cs_scratch);
  // forward-error estimate (sas.py:214-235)
  double cmax = 0.0, ymax = 0.0;
  for (int i = 0; i < m; ++i) {
    cmax = fmax(cmax, cabs2(c[i]));
    ymax = fmax(ymax, cabs2(y[i]));
  }
  const double denom = fmax(cmax, 1e-300);
  forward_apply(x, c, m, r);
  for (int j = 0; j < m; ++j) r[j] = cs(r[j], y[j]);
  vandermonde_solve_s(x, r, m, perm, d, cs_scratch);
  double dmax = 0.0;
  for (int i = 0; i < m; ++i) dmax = fmax(dmax, cabs2(d[i]));
  double est = dmax / denom;
  const double amp = a.node_amp[v];
  est = fmax(est, amp * noise_eps * ymax / denom);
  int flag = 0;
  double res = 0.0;
  if (!(est <= a.tol / 20.0)) {
    flag = 1;  // escalate to double-double
  } else {
    forward_apply(x, c, m, r);
    double num = 0.0, den = 0.0;
    for (int j = 0; j < m; ++j) {
      const C64x e = cs(r[j], y[j]);
      num += e.x * e.x + e.y * e.y;
      den += y[j].x * y[j].x + y[j].y * y[j].y;
    }
    res = sqrt(num) / fmax(sqrt(den), 1e-300);
    if (res > fmax(a.tol, 1e-9)) flag = 2;
  }
  for (int i = 0; i < m; ++i) out[a.node_mem[off + i]] = c[i];
  a.flags[fid] = flag;
  a.resid[fid] = res;
  if (flag == 1) a.esc_list[atomicAdd(&a.counts[0], 1u)] = (int32_t)fid;
  else if (flag == 2) a.fb_list[atomicAdd(&a.counts[1], 1u)] = (int32_t)fid;
}

// nodes heavier than kMaxMu (listed by k_sas_decode_f64): one CTA per item
__global__ void k_sas_decode_f64_big(const SasDecodeArgs a, const int32_t* __restrict__ work, int64_t n_work) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    if (threadIdx.x != 0) continue;
    const int64_t id = work[w];
    const int64_t b = id / a.n_nodes, v = id % a.n_nodes;
    const int off = a.node_off[v], m = a.node_off[v + 1] - off;
    C64x* x = reinterpret_cast<C64x*>(smem_raw);
    C64x* y = x + m;
    C64x* c = y + m;
    C64x* r = c + m;
    C64x* d = r + m;
    C64x* t = d + m;
    int* perm = reinterpret_cast<int*>(t + m);
    decode_node(a, b, v, off, m, x, y, c, r, d, t, perm);
  }
}

// one thread per (signal, node)
__global__ void k_sas_decode_f64(const SasDecodeArgs a) {
  const int64_t total = a.B * a.n_nodes;
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total;
       id += (int64_t)gridDim.x * blockDim.x) {
    // node-major: a warp decodes one node for 32 signals, so every lane runs
    // the same system size (node weights differ from node to node)
    const int64_t v = id / a.B, b = id % a.B;
    const int64_t fid = b * a.n_nodes + v;  // flags / resid stay (signal, node) row-major
    const int off = a.node_off[v], m = a.node_off[v + 1] - off;
    C64x* out = reinterpret_cast<C64x*>(a.out) + b * a.ld_out;
    if (m == 1) {
      const C64x raw = nodeval(a, b * a.mu, v);
      out[a.node_mem[off]] = a.scale == 1.0 ? raw : C64x{raw.x * a.scale, raw.y * a.scale};
      a.flags[fid] = 0;
      a.resid[fid] = 0.0;
      continue;
    }
    if (m > kMaxMu) {  // k_sas_decode_f64_big
      a.big_list[atomicAdd(&a.counts[2], 1u)] = (int32_t)fid;
      continue;
    }
    C64x x[kMaxMu], y[kMaxMu], c[kMaxMu], r[kMaxMu], d[kMaxMu], t[kMaxMu];
    int perm[kMaxMu];
    decode_node(a, b, v, off, m, x, y, c, r, d, t, perm);
  }
}

// --------------------------------------------- double-double escalation ---
struct SasDDArgs {
  SasDecodeArgs base;
  RootTab tab;
  const int64_t* pattern;  // sorted I_r, A entries
  int64_t A;
  const int32_t* node_res;  // residues (n_nodes)
  // samples: dense source (promoted) or precomputed dd samples (band-limited)
  const void* sig;
  int64_t ld_sig;
  int sig_c64;
  const cdd* samples_dd;  // (B x mu x A) at (pattern_i - j) mod N, or NULL
  const double2* table;   // same layout in float64 (callable sources), or NULL
  const int32_t* work;    // escalated (signal, node) ids
  int64_t n_work;
};

__device__ __forceinline__ cdd dd_sample(const SasDDArgs& a, int64_t b, int64_t j, int64_t i) {
  if (a.samples_dd) return a.samples_dd[(b * a.base.mu + j) * a.A + i];
  if (a.table) {
    const double2 v = a.table[(b * a.base.mu + j) * a.A + i];
    return {{v.x, 0.0}, {v.y, 0.0}};
  }
  const uint64_t loc = ((uint64_t)a.pattern[i] - (uint64_t)j) & a.tab.nmask;
  if (a.sig_c64) {
    const float2 v = reinterpret_cast<const float2*>(a.sig)[b * a.ld_sig + loc];
    return {{(double)v.x, 0.0}, {(double)v.y, 0.0}};
  }
  const double2 v = reinterpret_cast<const double2*>(a.sig)[b * a.ld_sig + loc];
  return {{v.x, 0.0}, {v.y, 0.0}};
}

__device__ __forceinline__ dd shfl_dd(dd v, int d) {
  return {__shfl_xor_sync(0xffffffffu, v.hi, d), __shfl_xor_sync(0xffffffffu, v.lo, d)};
}

// one WARP per escalated node: re-measure (sas.py:290-310) with the A-term dd
// dot products split across the lanes (butterfly-reduced in dd), then the
// warp solves in dd across its lanes (_ddc.py:235-254)
__global__ void k_sas_decode_dd(const SasDDArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < a.n_work; w += warps) {
    const int64_t id = a.work[w];
    const SasDecodeArgs& s = a.base;
    const int64_t b = id / s.n_nodes, v = id % s.n_nodes;
    const int off = s.node_off[v], m = s.node_off[v + 1] - off;
    if (m > kMaxMu) continue;  // k_sas_decode_dd_big
    const uint64_t resid = (uint64_t)(int64_t)a.node_res[v];
    cdd y[kMaxMu];
    // shifts in groups of JG: each root kernel value serves JG shifts (per
    // shift the lane still sums its terms in increasing i, as before)
    constexpr int JG = 4;
    for (int j0 = 0; j0 < m; j0 += JG) {
      cdd acc[JG];
#pragma unroll
      for (int g = 0; g < JG; ++g) acc[g] = {{0.0, 0.0}, {0.0, 0.0}};
      for (int64_t i = lane; i < a.A; i += 32) {
        const cdd kern = a.tab.get((uint64_t)(-(int64_t)(resid * (uint64_t)a.pattern[i])));
#pragma unroll
        for (int g = 0; g < JG; ++g)
          if (j0 + g < m) acc[g] = cdd_add(acc[g], cdd_mul(dd_sample(a, b, j0 + g, i), kern));
      }
#pragma unroll
      for (int g = 0; g < JG; ++g) {
        if (j0 + g >= m) break;
        cdd t = acc[g];
        for (int d = 16; d > 0; d >>= 1) {
          const cdd o = {shfl_dd(t.re, d), shfl_dd(t.im, d)};
          t = cdd_add(t, o);
        }
        y[j0 + g] = cdd_mul_complex(t, s.scale, 0.0);
      }
    }
    // solve_vandermonde_dd (x_m = root((-l) mod N), BP, no Leja), the lanes
    // holding the unknowns: inside each BP sweep every update reads only
    // values from before the sweep, so lane j (and j + 32) updates its own
    // entries from shuffled neighbours -- the same dd operations per entry as
    // the sequential loops, in the same order
    constexpr int Q = (kMaxMu + 31) / 32;
    cdd yl[Q], xl[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      yl[q] = j < m ? y[j] : cdd{{0.0, 0.0}, {0.0, 0.0}};
      xl[q] = j < m ? a.tab.get((uint64_t)(-(int64_t)s.J[s.node_mem[off + j]])) : cdd{{0.0, 0.0}, {0.0, 0.0}};
    }
    // value of entry j - 1 (dir -1) or j + 1 (dir +1) from before the sweep
    auto neighbour = [&](const cdd (&v)[Q], int q, int dir) -> cdd {
      const int src = (lane + dir) & 31;
      cdd r;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        const cdd t = {{__shfl_sync(0xffffffffu, v[qq].re.hi, src), __shfl_sync(0xffffffffu, v[qq].re.lo, src)},
                       {__shfl_sync(0xffffffffu, v[qq].im.hi, src), __shfl_sync(0xffffffffu, v[qq].im.lo, src)}};
        const int want = q + ((dir < 0 && lane == 0) ? -1 : (dir > 0 && lane == 31) ? 1 : 0);
        if (qq == want) r = t;
      }
      return r;
    };
    auto xat = [&](int idx) -> cdd {  // x[idx] broadcast from its lane
      cdd r = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        const cdd t = {{__shfl_sync(0xffffffffu, xl[qq].re.hi, idx & 31), __shfl_sync(0xffffffffu, xl[qq].re.lo, idx & 31)},
                       {__shfl_sync(0xffffffffu, xl[qq].im.hi, idx & 31), __shfl_sync(0xffffffffu, xl[qq].im.lo, idx & 31)}};
        if (qq == (idx >> 5)) r = t;
      }
      return r;
    };
    for (int k = 0; k < m - 1; ++k) {  // y[j] -= x[k] y[j-1], j = m-1 .. k+1
      const cdd xk = xat(k);
      cdd prev[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) prev[q] = neighbour(yl, q, -1);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = lane + 32 * q;
        if (j > k && j < m) yl[q] = cdd_sub(yl[q], cdd_mul(xk, prev[q]));
      }
    }
    for (int k = m - 2; k >= 0; --k) {
      // y[j] /= x[j] - x[j-k-1], j = k+1 .. m-1
      cdd xs[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = lane + 32 * q;
        const int src = j - k - 1;
        const cdd t = xat(src < 0 ? 0 : src);
        xs[q] = t;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = lane + 32 * q;
        if (j > k && j < m) yl[q] = cdd_div(yl[q], cdd_sub(xl[q], xs[q]));
      }
      // y[j] -= y[j+1], j = k .. m-2 (old y[j+1])
      cdd nxt[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) nxt[q] = neighbour(yl, q, +1);
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = lane + 32 * q;
        if (j >= k && j < m - 1) yl[q] = cdd_sub(yl[q], nxt[q]);
      }
    }
    C64x* out = reinterpret_cast<C64x*>(s.out) + b * s.ld_out;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      if (j < m)
        out[s.node_mem[off + j]] = {__dadd_rn(yl[q].re.hi, yl[q].re.lo), __dadd_rn(yl[q].im.hi, yl[q].im.lo)};
    }
  }
}

// escalation of nodes heavier than kMaxMu: one warp per node re-measures
// (the same lane-split dd dot products as k_sas_decode_dd), lane 0 solves in
// dd sequentially on shared memory -- the same operations per entry, in the
// same order, as the lane-parallel sweeps (_ddc.py:235-254)
__global__ void k_sas_decode_dd_big(const SasDDArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  for (int64_t w = blockIdx.x; w < a.n_work; w += gridDim.x) {
    const int64_t id = a.work[w];
    const SasDecodeArgs& s = a.base;
    const int64_t b = id / s.n_nodes, v = id % s.n_nodes;
    const int off = s.node_off[v], m = s.node_off[v + 1] - off;
    if (m <= kMaxMu) continue;
    cdd* y = reinterpret_cast<cdd*>(smem_raw);  // m
    cdd* xl = y + m;                              // m
    const uint64_t resid = (uint64_t)(int64_t)a.node_res[v];
    for (int j = 0; j < m; ++j) {
      cdd acc = {{0.0, 0.0}, {0.0, 0.0}};
      for (int64_t i = lane; i < a.A; i += 32) {
        const cdd kern = a.tab.get((uint64_t)(-(int64_t)(resid * (uint64_t)a.pattern[i])));
        acc = cdd_add(acc, cdd_mul(dd_sample(a, b, j, i), kern));
      }
      for (int d = 16; d > 0; d >>= 1) {
        const cdd o = {shfl_dd(acc.re, d), shfl_dd(acc.im, d)};
        acc = cdd_add(acc, o);
      }
      if (lane == 0) y[j] = cdd_mul_complex(acc, s.scale, 0.0);
    }
    for (int j = lane; j < m; j += 32) xl[j] = a.tab.get((uint64_t)(-(int64_t)s.J[s.node_mem[off + j]]));
    __syncwarp();
    if (lane == 0) {
      for (int k = 0; k < m - 1; ++k)
        for (int j = m - 1; j > k; --j) y[j] = cdd_sub(y[j], cdd_mul(xl[k], y[j - 1]));
      for (int k = m - 2; k >= 0; --k) {
        for (int j = k + 1; j < m; ++j) y[j] = cdd_div(y[j], cdd_sub(xl[j], xl[j - k - 1]));
        for (int j = k; j < m - 1; ++j) y[j] = cdd_sub(y[j], y[j + 1]);
      }
      C64x* out = reinterpret_cast<C64x*>(s.out) + b * s.ld_out;
      for (int j = 0; j < m; ++j)
        out[s.node_mem[off + j]] = {__dadd_rn(y[j].re.hi, y[j].re.lo), __dadd_rn(y[j].im.hi, y[j].im.lo)};
    }
    __syncwarp();
  }
}

// band-limited source: dd samples at (pattern_i - j) mod N for j < mu (synthesize_dd, _ddc.py:212-224)
__global__ void k_dd_samples(RootTab tab, const int64_t* __restrict__ pattern, int64_t A, int64_t mu,
                             const int64_t* __restrict__ Jsrc, const double2* __restrict__ csrc, int64_t ksrc,
                             int M, const int32_t* __restrict__ sigs, int64_t nsig, cdd* __restrict__ out) {
  const int64_t total = nsig * mu * A;
  const double invN = ldexp(1.0, -M);
  for (int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; id < total; id += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = id % A, j = (id / A) % mu, sidx = id / (A * mu);
    const int64_t bsig = sigs[sidx];
    const uint64_t loc = ((uint64_t)pattern[i] - (uint64_t)j) & tab.nmask;
    const int64_t* Jb = Jsrc;
    const double2* cb = csrc + bsig * ksrc;
    cdd acc = {{0.0, 0.0}, {0.0, 0.0}};
    for (int64_t e = 0; e < ksrc; ++e)
      acc = cdd_add(acc, cdd_mul_complex(tab.get(loc * (uint64_t)Jb[e]), cb[e].x, cb[e].y));
    out[(bsig * mu + j) * A + i] = cdd_mul_complex(acc, invN, 0.0);
  }
}

// dense fallback (sas.py:389-395): LU with partial pivoting of V (V[j][m] = x_m^j)
__device__ void dense_node(const SasDecodeArgs& a, int64_t b, int64_t v, int off, int m, C64x* V, C64x* rhs, C64x* x,
                           C64x* sol) {
  const double N = ldexp(1.0, a.M);
  for (int i = 0; i < m; ++i) {
    double sn, co;
    sincospi(-2.0 * (double)a.J[a.node_mem[off + i]] / N, &sn, &co);
    x[i] = {co, sn};
  }
  for (int j = 0; j < m; ++j) {
    const C64x raw = nodeval(a, b * a.mu + j, v);
    rhs[j] = {raw.x * a.scale, raw.y * a.scale};
    for (int i = 0; i < m; ++i) {
      C64x p = {1.0, 0.0};
      for (int e = 0; e < j; ++e) p = cm(p, x[i]);
      V[j * m + i] = p;
    }
  }
  for (int col = 0; col < m; ++col) {
    int piv = col;
    double best = cabs2(V[col * m + col]);
    for (int r = col + 1; r < m; ++r)
      if (cabs2(V[r * m + col]) > best) { best = cabs2(V[r * m + col]); piv = r; }
    if (piv != col) {
      for (int c2 = 0; c2 < m; ++c2) {
        const C64x t = V[col * m + c2];
        V[col * m + c2] = V[piv * m + c2];
        V[piv * m + c2] = t;
      }
      const C64x t = rhs[col];
      rhs[col] = rhs[piv];
      rhs[piv] = t;
    }
    for (int r = col + 1; r < m; ++r) {
      const C64x f = cdv(V[r * m + col], V[col * m + col]);
      for (int c2 = col; c2 < m; ++c2) V[r * m + c2] = cs(V[r * m + c2], cm(f, V[col * m + c2]));
      rhs[r] = cs(rhs[r], cm(f, rhs[col]));
    }
  }
  C64x* out = reinterpret_cast<C64x*>(a.out) + b * a.ld_out;
  for (int r = m - 1; r >= 0; --r) {
    C64x acc = rhs[r];
    for (int c2 = r + 1; c2 < m; ++c2) acc = cs(acc, cm(V[r * m + c2], sol[c2]));
    sol[r] = cdv(acc, V[r * m + r]);
  }
  for (int i = 0; i < m; ++i) out[a.node_mem[off + i]] = sol[i];
}

__global__ void k_sas_dense(const SasDecodeArgs a, const int32_t* __restrict__ work, int64_t n_work,
                            C64x* __restrict__ scratch) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n_work; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t id = work[w];
    const int64_t b = id / a.n_nodes, v = id % a.n_nodes;
    const int off = a.node_off[v], m = a.node_off[v + 1] - off;
    if (m > kMaxMu) continue;  // k_sas_dense_big
    C64x rhs[kMaxMu], x[kMaxMu], sol[kMaxMu];
    dense_node(a, b, v, off, m, scratch + w * kMaxMu * kMaxMu, rhs, x, sol);
  }
}

// dense fallback for nodes heavier than kMaxMu: one CTA per item, thread 0,
// vectors in shared memory, V (mu x mu) in global scratch
__global__ void k_sas_dense_big(const SasDecodeArgs a, const int32_t* __restrict__ work, int64_t n_work,
                                C64x* __restrict__ scratch, int64_t mu) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  for (int64_t w = blockIdx.x; w < n_work; w += gridDim.x) {
    if (threadIdx.x != 0) continue;
    const int64_t id = work[w];
    const int64_t b = id / a.n_nodes, v = id % a.n_nodes;
    const int off = a.node_off[v], m = a.node_off[v + 1] - off;
    if (m <= kMaxMu) continue;
    C64x* rhs = reinterpret_cast<C64x*>(smem_raw);
    dense_node(a, b, v, off, m, scratch + blockIdx.x * mu * mu, rhs, rhs + m, rhs + 2 * m);
  }
}

// node membership in CSR form, members ascending (deterministic: per round
// every node claims its smallest unclaimed member)
__global__ void k_node_counts(const int32_t* __restrict__ slot_count_src, const int32_t* __restrict__ node_slots,
                              int64_t n_nodes, int32_t* __restrict__ off) {
  // single CTA exclusive scan of the node weights
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < n_nodes; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    __shared__ int32_t buf[1024];
    buf[threadIdx.x] = i < n_nodes ? slot_count_src[node_slots[i]] : 0;
    __syncthreads();
    for (int d = 1; d < (int)blockDim.x; d <<= 1) {
      const int32_t add = threadIdx.x >= (unsigned)d ? buf[threadIdx.x - d] : 0;
      __syncthreads();
      buf[threadIdx.x] += add;
      __syncthreads();
    }
    const int32_t incl = buf[threadIdx.x];
    const int32_t c0 = carry;
    const int32_t w = i < n_nodes ? slot_count_src[node_slots[i]] : 0;
    if (i < n_nodes) off[i] = c0 + incl - w;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c0 + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[n_nodes] = carry;
}

__global__ void k_slot_counts(const int32_t* __restrict__ pats, int64_t k, int32_t* __restrict__ count) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&count[pats[e]], 1);
}

__global__ void k_member_round(const int32_t* __restrict__ pats, const int32_t* __restrict__ inv_node, int64_t k,
                               uint8_t* __restrict__ taken, int32_t* __restrict__ cand) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < k; e += (int64_t)gridDim.x * blockDim.x)
    if (!taken[e]) atomicMin(&cand[inv_node[pats[e]]], (int32_t)e);
}
__global__ void k_member_take(int32_t* __restrict__ cand, const int32_t* __restrict__ off, int64_t n_nodes, int round,
                              uint8_t* __restrict__ taken, int32_t* __restrict__ mem) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n_nodes; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = cand[v];
    if (e != 0x7fffffff) {
      mem[off[v] + round] = e;
      taken[e] = 1;
      cand[v] = 0x7fffffff;
    }
  }
}

__global__ void k_fill_i32(int32_t* __restrict__ p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

static int grid_for(int64_t n, int threads);

// double-double root tables per (device, M), built once (the reference caches
// its RootTable per modulus too, _ddc.py:208-209)
static std::mutex g_root_mu;
static std::map<std::pair<int, int>, std::pair<cdd*, cdd*>> g_roots;

static int root_tables(int M, cdd** fine, cdd** coarse, cudaStream_t st) {
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_root_mu);
  auto it = g_roots.find({dev, M});
  if (it == g_roots.end()) {
    const int h = M / 2;
    cdd *f = nullptr, *c = nullptr;
    SFFT_CUDA(cudaMalloc(&f, sizeof(cdd) * (1ll << h)));
    SFFT_CUDA(cudaMalloc(&c, sizeof(cdd) * (1ll << (M - h))));
    k_root_tables<<<grid_for((1ll << h) + (1ll << (M - h)), 128), 128, 0, st>>>(f, c, M);
    SFFT_CUDA(cudaGetLastError());
    SFFT_CUDA(cudaStreamSynchronize(st));  // usable from any stream afterwards
    it = g_roots.emplace(std::make_pair(dev, M), std::make_pair(f, c)).first;
  }
  *fine = it->second.first;
  *coarse = it->second.second;
  return SFFT_OK;
}

static int grid_for(int64_t n, int threads = 128) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)num_sms() * 32));
}

}  // namespace sfft

using namespace sfft;

// node CSR (offsets n_nodes+1, members k) for a plan; cached on the plan
static std::mutex g_nodes_mu;

extern "C" int sfft_plan_nodes(sfft_plan* p, int32_t* off_out, int32_t* mem_out, sfft_stream_t stream) {
  SFFT_NVTX("sfft_plan_nodes");
  cudaStream_t st = (cudaStream_t)stream;
  if (!p) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(p, "sfft_plan_nodes")) return rj;
  std::lock_guard<std::mutex> lk(g_nodes_mu);  // the table is built once, lazily
  if (!p->d_node_off) {
    int32_t *cnt = nullptr, *cand = nullptr;
    uint8_t* taken = nullptr;
    SFFT_CUDA(cudaMalloc(&p->d_node_off, 4 * (p->n_nodes + 1)));
    SFFT_CUDA(cudaMalloc(&p->d_node_mem, 4 * std::max<int64_t>(p->k, 1)));
    SFFT_CUDA(cudaMallocAsync(&cnt, 4 * p->A, st));
    SFFT_CUDA(cudaMallocAsync(&cand, 4 * std::max<int64_t>(p->n_nodes, 1), st));
    SFFT_CUDA(cudaMallocAsync(&taken, std::max<int64_t>(p->k, 1), st));
    SFFT_CUDA(cudaMemsetAsync(cnt, 0, 4 * p->A, st));
    k_fill_i32<<<grid_for(p->n_nodes), 128, 0, st>>>(cand, p->n_nodes, 0x7fffffff);
    SFFT_CUDA(cudaMemsetAsync(taken, 0, p->k, st));
    k_slot_counts<<<grid_for(p->k, 256), 256, 0, st>>>(p->d_element_slots, p->k, cnt);
    k_node_counts<<<1, 1024, 0, st>>>(cnt, p->d_node_slots, p->n_nodes, p->d_node_off);
    for (int64_t round = 0; round < p->mu_star; ++round) {
      k_member_round<<<grid_for(p->k, 256), 256, 0, st>>>(p->d_element_slots, p->d_inv_node, p->k, taken, cand);
      k_member_take<<<grid_for(p->n_nodes), 128, 0, st>>>(cand, p->d_node_off, p->n_nodes, (int)round, taken,
                                                          p->d_node_mem);
    }
    SFFT_CUDA(cudaGetLastError());
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(cand, st);
    cudaFreeAsync(taken, st);
  }
  if (off_out) SFFT_CUDA(cudaMemcpyAsync(off_out, p->d_node_off, 4 * (p->n_nodes + 1), cudaMemcpyDefault, st));
  if (mem_out) SFFT_CUDA(cudaMemcpyAsync(mem_out, p->d_node_mem, 4 * p->k, cudaMemcpyDefault, st));
  if (off_out || mem_out) SFFT_CUDA(cudaStreamSynchronize(st));
  return SFFT_OK;
}

// the mu* shifted Hi-DFTs of sas.py:343-345 in one launch: rows b*nshift + j
extern "C" int sfft_hidft_shifts(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int in_dtype,
                                 int64_t shift0, int64_t nshift, int out_kind, void* out, int64_t ld_out,
                                 sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_shifts");
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(plan, "sfft_hidft_shifts")) return rj;
  if (nshift < 1) return fail(SFFT_ERR_INVALID, "nshift must be >= 1");
  if (in_dtype != plan->dtype && !(in_dtype == SFFT_C64 && plan->dtype == SFFT_C128))
    return fail(SFFT_ERR_INVALID, "complex128 signals need a complex128 plan");
  if (B == 0) return SFFT_OK;
  const int32_t *map = nullptr, *inv = nullptr;
  int64_t n_out = 0;
  double scale = 1.0;
  int rc = out_spec(plan, out_kind, &map, &n_out, &scale, &inv);
  if (rc) return rc;
  if (ld < (1ll << plan->M) || ld_out < n_out) return fail(SFFT_ERR_INVALID, "row stride too small");
  return launch_hidft_plan(plan, signals, B, ld, shift0, map, inv, n_out, scale, out, ld_out, nullptr, 0, 0,
                           (cudaStream_t)stream, nshift, in_dtype != plan->dtype);
}

// decode: nodevals (B*mu rows) -> out (B x k complex128); flags/resid per (signal, node).
// source for escalation: dense signals (sig, ld_sig, sig_dtype) or, when
// bl_J != NULL, band-limited spectra (bl_J[k_src], bl_c[B x k_src] complex128).
// Returns counts through n_escalated / n_fallback.
extern "C" int sfft_sas_decode(sfft_plan* p, const void* nodevals, int64_t ld_nv, int nv_dtype, int64_t B,
                               int64_t mu, double tol, const void* sig, int64_t ld_sig, int sig_dtype,
                               const void* table, const int64_t* bl_J, const void* bl_c, int64_t k_src,
                               const int64_t* J_dev,
                               void* out, int64_t ld_out, int32_t* flags, double* resid, int64_t* n_escalated,
                               int64_t* n_fallback, sfft_stream_t stream) {
  SFFT_NVTX("sfft_sas_decode");
  cudaStream_t st = (cudaStream_t)stream;
  if (!p) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(p, "sfft_sas_decode")) return rj;
  if (p->height != 0) return fail(SFFT_ERR_CONTRACT, "sas decode needs height 0");
  if (mu != p->mu_star) return fail(SFFT_ERR_INVALID, "mu must equal the plan's mu*");
  if (mu > kMaxMuBig) return fail(SFFT_ERR_UNSUPPORTED, "node weight above " + std::to_string(kMaxMuBig));
  int rc = sfft_plan_nodes(p, nullptr, nullptr, stream);
  if (rc) return rc;
  if (!J_dev) return fail(SFFT_ERR_INVALID, "null support pointer");
  {  // signal-independent node tables, built once per plan
    std::lock_guard<std::mutex> lk(g_nodes_mu);
    if (!p->d_node_amp) {
      SFFT_CUDA(cudaMalloc(&p->d_node_x, sizeof(C64x) * std::max<int64_t>(p->k, 1)));
      SFFT_CUDA(cudaMalloc((void**)&p->d_node_perm, sizeof(int32_t) * std::max<int64_t>(p->k, 1)));
      SFFT_CUDA(cudaMalloc((void**)&p->d_node_amp, sizeof(double) * std::max<int64_t>(p->n_nodes, 1)));
      k_node_prep<<<grid_for(p->n_nodes, 128), 128, 0, st>>>(p->d_node_off, p->d_node_mem, J_dev, p->n_nodes, p->M,
                                                             (C64x*)p->d_node_x, p->d_node_perm, p->d_node_amp);
      if (mu > kMaxMu) {
        const size_t sm = (2 * mu + 1) * sizeof(C64x) + mu * (sizeof(double) + sizeof(int) + 1);
        SFFT_CUDA(cudaFuncSetAttribute(k_node_prep_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_node_prep_big<<<(unsigned)std::min<int64_t>(p->n_nodes, (int64_t)num_sms() * 8), 32, sm, st>>>(
            p->d_node_off, p->d_node_mem, J_dev, p->n_nodes, p->M, (C64x*)p->d_node_x, p->d_node_perm,
            p->d_node_amp);
      }
      SFFT_CUDA(cudaGetLastError());
    }
  }
  SasDecodeArgs a{};
  a.nodevals = nodevals;
  a.ld_nv = ld_nv;
  a.nv_c64 = nv_dtype == SFFT_C64;
  a.B = B;
  a.mu = mu;
  a.n_nodes = p->n_nodes;
  a.k = p->k;
  a.M = p->M;
  a.scale = ldexp(1.0, p->M) / (double)p->A;
  a.tol = tol;
  a.node_off = p->d_node_off;
  a.node_mem = p->d_node_mem;
  a.J = J_dev;
  a.out = out;
  a.ld_out = ld_out;
  a.flags = flags;
  a.resid = resid;
  a.node_x = (const C64x*)p->d_node_x;
  a.node_perm = p->d_node_perm;
  a.node_amp = p->d_node_amp;
  // escalation / fallback work lists compacted on the device: only their
  // lengths come back to the host
  const int64_t total = B * p->n_nodes;
  int32_t* lists = nullptr;
  SFFT_CUDA(cudaMallocAsync((void**)&lists, sizeof(int32_t) * (3 * total + 3), st));
  a.esc_list = lists;
  a.fb_list = lists + total;
  a.big_list = lists + 2 * total;
  a.counts = reinterpret_cast<unsigned int*>(lists + 3 * total);
  SFFT_CUDA(cudaMemsetAsync(a.counts, 0, 3 * sizeof(unsigned int), st));
  k_sas_decode_f64<<<grid_for(total), 128, 0, st>>>(a);
  SFFT_CUDA(cudaGetLastError());
  unsigned int hc[3] = {0, 0, 0};
  SFFT_CUDA(cudaMemcpyAsync(hc, a.counts, sizeof(hc), cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  if (hc[2] > 0) {  // nodes heavier than kMaxMu: one CTA each
    const size_t sm = 6 * mu * sizeof(C64x) + mu * sizeof(int);
    SFFT_CUDA(cudaFuncSetAttribute(k_sas_decode_f64_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_sas_decode_f64_big<<<(unsigned)std::min<int64_t>(hc[2], (int64_t)num_sms() * 8), 32, sm, st>>>(
        a, a.big_list, (int64_t)hc[2]);
    SFFT_CUDA(cudaGetLastError());
    SFFT_CUDA(cudaMemcpyAsync(hc, a.counts, 2 * sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    SFFT_CUDA(cudaStreamSynchronize(st));
  }
  const int64_t n_esc = hc[0], n_fb = hc[1];
  *n_escalated = n_esc;
  *n_fallback = n_fb;
  if (n_esc > 0) {
    const int M = p->M, h = M / 2;
    cdd *fine = nullptr, *coarse = nullptr, *samples = nullptr;
    if ((rc = root_tables(M, &fine, &coarse, st))) return rc;
    int64_t* pattern = nullptr;
    int32_t* sigs = nullptr;
    SFFT_CUDA(cudaMallocAsync(&pattern, 8 * p->A, st));
    rc = sfft_pivoted_pattern(p->used, p->s, M, pattern, stream);
    if (rc) return rc;
    SasDDArgs d{};
    d.base = a;
    d.tab = RootTab{fine, coarse, h, (1ull << M) - 1};
    d.pattern = pattern;
    d.A = p->A;
    d.node_res = p->d_node_residues;
    d.sig = sig;
    d.ld_sig = ld_sig;
    d.sig_c64 = sig_dtype == SFFT_C64;
    d.table = (const double2*)table;
    d.work = a.esc_list;
    d.n_work = n_esc;
    if (bl_J) {  // band-limited: dd samples for the signals that escalated
      std::vector<int32_t> esc((size_t)n_esc);
      SFFT_CUDA(cudaMemcpyAsync(esc.data(), a.esc_list, 4 * esc.size(), cudaMemcpyDeviceToHost, st));
      SFFT_CUDA(cudaStreamSynchronize(st));
      std::vector<int32_t> s2;
      for (int32_t id : esc) s2.push_back((int32_t)(id / p->n_nodes));
      std::sort(s2.begin(), s2.end());
      s2.erase(std::unique(s2.begin(), s2.end()), s2.end());
      SFFT_CUDA(cudaMallocAsync(&sigs, 4 * s2.size(), st));
      SFFT_CUDA(cudaMemcpyAsync(sigs, s2.data(), 4 * s2.size(), cudaMemcpyHostToDevice, st));
      SFFT_CUDA(cudaMallocAsync(&samples, sizeof(cdd) * B * mu * p->A, st));
      k_dd_samples<<<grid_for((int64_t)s2.size() * mu * p->A), 128, 0, st>>>(
          d.tab, pattern, p->A, mu, bl_J, (const double2*)bl_c, k_src, M, sigs, (int64_t)s2.size(), samples);
      d.samples_dd = samples;
    }
    k_sas_decode_dd<<<grid_for(d.n_work * 32, 128), 128, 0, st>>>(d);
    if (mu > kMaxMu) {
      const size_t sm = 2 * mu * sizeof(cdd);
      SFFT_CUDA(cudaFuncSetAttribute(k_sas_decode_dd_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_sas_decode_dd_big<<<(unsigned)std::min<int64_t>(d.n_work, (int64_t)num_sms() * 8), 32, sm, st>>>(d);
    }
    SFFT_CUDA(cudaGetLastError());
    cudaFreeAsync(pattern, st);
    if (sigs) cudaFreeAsync(sigs, st);
    if (samples) cudaFreeAsync(samples, st);
  }
  if (n_fb > 0) {
    C64x* scratch = nullptr;
    SFFT_CUDA(cudaMallocAsync(&scratch, sizeof(C64x) * kMaxMu * kMaxMu * n_fb, st));
    k_sas_dense<<<grid_for(n_fb, 32), 32, 0, st>>>(a, a.fb_list, n_fb, scratch);
    SFFT_CUDA(cudaGetLastError());
    cudaFreeAsync(scratch, st);
    if (mu > kMaxMu) {
      const int64_t g = std::min<int64_t>(n_fb, (int64_t)num_sms() * 2);
      C64x* big = nullptr;
      SFFT_CUDA(cudaMallocAsync(&big, sizeof(C64x) * mu * mu * g, st));
      const size_t sm = 3 * mu * sizeof(C64x);
      SFFT_CUDA(cudaFuncSetAttribute(k_sas_dense_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_sas_dense_big<<<(unsigned)g, 32, sm, st>>>(a, a.fb_list, n_fb, big, mu);
      SFFT_CUDA(cudaGetLastError());
      cudaFreeAsync(big, st);
    }
  }
  cudaFreeAsync(lists, st);
  return SFFT_OK;
}
