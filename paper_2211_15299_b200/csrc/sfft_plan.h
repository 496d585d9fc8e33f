// Internal plan object shared by the plan builder and the transform launchers.
#pragma once

#include <stdint.h>

#include <utility>

struct sfft_plan {
  int device;
  int M, dtype, n_r, height, s, level, homogeneous;
  int64_t k, A, n_nodes, mu_star;
  uint64_t pivot_mask;
  int32_t r[32];
  int32_t used[32];
  // device tables (int32 indices: N <= 2^31)
  int32_t* d_element_slots;  // k   slot of each support element (pats)
  int32_t* d_slot_residues;  // A   residue mod 2^level, virtual slots inherit
  uint8_t* d_slot_real;      // A
  int32_t* d_node_slots;     // n_nodes  real slots in ascending residue order
  int32_t* d_node_residues;  // n_nodes
  void* d_twiddles;          // A-1 complex (dtype), stage-major
  int32_t* d_inv_elem;       // A   slot -> support element (-1: virtual); unique when mu* = 1
  int32_t* d_inv_node;       // A   slot -> node rank (-1: virtual)
  int32_t* d_node_off;       // n_nodes+1  node membership CSR (built on first SAS decode)
  int32_t* d_node_mem;       // k          member element indices, ascending per node
  void* d_node_x;            // k complex128: e^{-2 pi i J/N} per member (SAS decode, built on first use)
  int32_t* d_node_perm;      // k          Leja order within each node
  double* d_node_amp;        // n_nodes    ||inv(V)||_inf per node
  // two-pass (split) transform for 2^s beyond one CTA (sfft_hidft.cu, k_split_*):
  // block t of 2^lc holds the slots whose low lc bits are brev_lc(t)
  int split_lc;              // lc (0: single-CTA plan)
  void* d_tw_blk;            // 2^lc x (2^(s-lc) - 1) twiddles of the local stages, per block, stage-major
  int32_t* d_inv_elem_blk;   // A   d_inv_elem, block-major: [t][l] = inv_elem[(l << lc) | brev_lc(t)]
  int32_t* d_inv_node_blk;   // A   d_inv_node, block-major
  // three-pass split (sfft_split.cu, k_tri_*): slot = (b << (s-4)) | q; the
  // final pass owns the q of one position pi = rank of q in d_tri_perm order
  int32_t* d_tri_perm;       // 2^(s-4)  pi -> q, sorted by mean output position
  int32_t* d_tri_pinv;       // 2^(s-4)  q -> pi (the head pass's bulk epilogue stores position pi)
  void* d_tri_tw;            // 15 x 2^(s-4) twiddles of the last 4 stages, [j][pi]
  int32_t* d_tri_inv_elem;   // 16 x 2^(s-4)  [b][pi] = d_inv_elem[(b << (s-4)) | perm[pi]]
  int32_t* d_tri_inv_node;   // 16 x 2^(s-4)  same for d_inv_node
  unsigned char tri_front_tw[16 * 31];  // host copy of twiddles 0..30 (stages 1..5), plan dtype
  // complex64 middle pass: shared-memory positions of its last stores and of
  // the permuted epilogue reads, chosen so both are bank-conflict free
  int32_t* d_tri_spos;       // 2^(s-4)  [x][tid] -> position of the value thread tid stores from register x
  int32_t* d_tri_ppos;       // 2^(s-4)  [pi] -> position of q = perm[pi]
  // the same for the head pass's last register pass and epilogue (k_head)
  int32_t* d_head_spos;      // 2^(s-4)  [x][tt] -> position of the value thread tt stores from register x
  int32_t* d_head_ppos;      // 2^(s-4)  [pi] -> position of q = perm[pi]
  // the final pass's output map is blocked: d_tri_inv_*[b][pi] = T * 2^(s-4) + pi
  // for a per-pi bijection b -> T (coalesced staged stores, sfft_split.cu k_fin2)
  int tri_blocked_elem, tri_blocked_node;
  // per-signal supports (sfft_plan_batched): tables derived on chip per signal
  int per_signal;
  int64_t n_supports;
  int64_t* d_J;              // n_supports x k
};

namespace sfft {
// largest s handled on one CTA (one signal's slots resident in shared memory)
constexpr int kMaxPlanS_c64 = 14, kMaxPlanS_c128 = 13;
// largest s of the fused per-signal transform (plan derived on chip)
constexpr int kMaxFusedS_c64 = 13, kMaxFusedS_c128 = 12;
// largest s of the device transform (two-pass split beyond kMaxPlanS)
constexpr int kMaxSplitS_c64 = 17, kMaxSplitS_c128 = 16;
// split for 2^s beyond one CTA: the first lc stages run across 2^lc blocks,
// the remaining s - lc (12, or 13 for s = 17) inside one CTA per block
inline int split_lc(int dtype, int s) {
  if (dtype == SFFT_C64) return (s > kMaxPlanS_c64 && s <= kMaxSplitS_c64) ? (s == 17 ? 4 : s - 12) : 0;
  return (s > kMaxPlanS_c128 && s <= kMaxSplitS_c128) ? s - 12 : 0;
}
// transform launchers (sfft_hidft.cu)
int launch_hidft_plan(const sfft_plan* p, const void* sig, int64_t B, int64_t ld, int64_t shift,
                      const int32_t* map1, const int32_t* inv1, int64_t n1, double scale1, void* out1,
                      int64_t ld1, void* out2, int64_t ld2, int identity, cudaStream_t st,
                      int64_t nshift = 1, int in_c64 = 0);
int max_supported_s(int dtype);
// programmatic-dependent-launch chain of one stream (sfft_hidft.cu): true if
// a launch reading `in` may overlap the chain's running launches; records
// its outputs (or restarts the chain when it must launch fully ordered)
using ByteRange = std::pair<uintptr_t, uintptr_t>;
bool pdl_join(cudaStream_t st, const ByteRange* in, int nin, const ByteRange* out, int nout, bool eligible);
// device-resident transforms of this plan take the TMA head path (sfft_split.cu)
bool head_covers(const sfft_plan* p);
// SFFT_SPLIT_PASSES=2: the two-pass split (its block-major tables are built only then)
bool split_two_pass();
// per-signal plans only serve sfft_hidft(SFFT_OUT_DFT)
int reject_per_signal(const sfft_plan* p, const char* entry);
// hidft_to_dft for per-signal supports (sfft_hidft_to_dft_fused's body)
// identity: rows pre-gathered in each row's own slot order (row stride >= k)
int fused_to_dft(const int64_t* J, int64_t k, int64_t n_supports, int M, const void* signals, int64_t B,
                 int64_t ld, int dtype, void* out, int64_t ld_out, int32_t* status, cudaStream_t st,
                 int identity = 0);
// pre-gathered rows (identity loads): slot order, or sorted order when
// gathered_sorted(plan) (the cluster transform, 2^s beyond one CTA)
bool gathered_sorted(const sfft_plan* p);
int hidft_gathered(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld, int sorted, int out_kind,
                   void* out, int64_t ld_out, void* slot_out, int64_t ld_slot, cudaStream_t st);
int out_spec(const sfft_plan* plan, int out_kind, const int32_t** map, int64_t* n_out, double* scale,
             const int32_t** inv = nullptr);
}  // namespace sfft
