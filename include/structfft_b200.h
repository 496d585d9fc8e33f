/*
 * structfft_b200.h -- C-ABI of the B200-native Hi-DFT (arXiv 2211.15299).
 *
 * Plain C: pointers, sizes, status codes, an opaque plan handle and a raw
 * cudaStream_t.  No torch types.  Every entry point replaces one function of
 * the reference Python package `structfft` (paths relative to
 * /root/reference/pkg/src/structfft); INTEGRATION.md shows the ctypes binding.
 *
 * Conventions (core.py:3-6): forward kernel e^{-2 pi i m n / N}; a shift a
 * reads the samples at (I - a) mod N; hidft output is the UNSCALED product
 * F(J, I) f_I; the DFT epilogue multiplies by N/|J| (hidft.py:188-207).
 *
 * Status codes mirror the reference exception classes and the CLI exit codes
 * (errors.py:4-17, cli.py:366-378): 0 ok, 2 InvalidInputError,
 * 3 ContractViolationError, 4 BudgetExceededError.  5 = CUDA runtime error,
 * 6 = size outside the device path.  The message of the last
 * failing call on the calling thread is available from sfft_last_error().
 *
 * Pointers: support indices J may be host or device memory (detected with
 * cudaPointerGetAttributes).  Signals may be device memory or page-locked
 * host memory mapped into the device address space (zero-copy gather).
 * Outputs are device (or mapped host) memory owned by the caller.
 * All calls are stream-ordered on `stream` and deterministic (no atomics in
 * the arithmetic).
 */
#ifndef STRUCTFFT_B200_H
#define STRUCTFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SFFT_API __attribute__((visibility("default")))
#else
#define SFFT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* sfft_stream_t; /* == cudaStream_t */

enum sfft_status {
  SFFT_OK = 0,
  SFFT_ERR_INVALID = 2,    /* errors.py:8  InvalidInputError       */
  SFFT_ERR_CONTRACT = 3,   /* errors.py:12 ContractViolationError  */
  SFFT_ERR_BUDGET = 4,     /* errors.py:16 BudgetExceededError     */
  SFFT_ERR_CUDA = 5,
  SFFT_ERR_UNSUPPORTED = 6
};

enum sfft_dtype { SFFT_C64 = 0, SFFT_C128 = 1 };

/* what the transform writes per signal row */
enum sfft_out_kind {
  SFFT_OUT_NODES = 0, /* HiDftResult.node_values, ascending node residue (hidft.py:168-178) */
  SFFT_OUT_DFT = 1,   /* hidft_to_dft: ascending-J order x N/|J| (hidft.py:188-207)          */
  SFFT_OUT_SAS = 2,   /* sas_transform mu*=1: ascending-J order x N/|I| (sas.py:358-371)     */
  SFFT_OUT_SLOTS = 3  /* HiDftResult.slot_values, slot order (hidft.py:180)                   */
};

/* layout of pre-gathered sample rows (A = 2^s per row) */
enum sfft_sample_order {
  SFFT_ORDER_SLOT = 0,    /* row[a] = f(off(a) - shift), slot order (hidft.py:155-158)          */
  SFFT_ORDER_PATTERN = 1  /* row[q] = f(I_r[q] - shift), ascending pattern (pivoted_pattern)    */
};

SFFT_API const char* sfft_version(void);
SFFT_API const char* sfft_last_error(void);
/* 1 if the library was compiled for and can run on the current device */
SFFT_API int sfft_device_ok(void);

/* pivots(J) -> bit mask of pivot levels, and classify(J) homogeneity.
 * Replaces congruence.py:76-101 (pivots) and congruence.py:235-241 (classify).
 * J: k strictly increasing indices in [0, 2^M), 1 <= M <= 31. */
SFFT_API int sfft_analyze(const int64_t* J, int64_t k, int M, uint64_t* pivot_mask,
                 int* homogeneous, sfft_stream_t stream);

/* pivoted_pattern(r, M).samples (sampling.py:62-71): the 2^n_r elements of
 * I_r in ascending order, written to `out` (host or device int64). */
SFFT_API int sfft_pivoted_pattern(const int32_t* r, int n_r, int M, int64_t* out,
                         sfft_stream_t stream);

typedef struct sfft_plan sfft_plan;

typedef struct sfft_plan_info {
  int M;               /* log2 N                                   */
  int dtype;           /* SFFT_C64 / SFFT_C128                     */
  int n_r;             /* len(r)                                   */
  int height;          /* n                                        */
  int s;               /* pivots merged by the butterfly           */
  int level;           /* output nodes live at this tree level     */
  int homogeneous;     /* classify(J).is_homogeneous               */
  int per_signal;      /* 1: sfft_plan_batched plan (one support per signal) */
  int64_t k;           /* |J|                                      */
  int64_t A;           /* 2^s slots = |I|                          */
  int64_t n_nodes;     /* real slots = nodes at `level`            */
  int64_t mu_star;     /* max node weight at `level` (sas.py:73-76)*/
  uint64_t pivot_mask; /* pivots(J)                                */
  int32_t used[32];    /* r[:n_r-height]                           */
} sfft_plan_info;

/* ButterflyPlan for (J, r, height): the checks of hidft.py:149-153
 * (validate_pivot_vector, assert_part_homogeneous, height range) and the
 * tables of _build_plan (hidft.py:69-95), built on the device.  Contract
 * failures return SFFT_ERR_CONTRACT with the offending pivot in the message. */
SFFT_API int sfft_plan_create(const int64_t* J, int64_t k, int M, const int32_t* r, int n_r,
                     int height, int dtype, sfft_stream_t stream, sfft_plan** plan);

/* Plan for PER-SIGNAL supports (config 4): n_supports rows of k indices
 * (int64, host or device, each a valid homogeneous SupportSet of Z_{2^M},
 * k = 2^s).  Nothing is derived on the host: pivots, pattern, tables and
 * twiddles of each support are built on chip by the transform (the fused
 * kernel of sfft_hidft_to_dft_fused).  Such a plan serves sfft_hidft with
 * SFFT_OUT_DFT, shift 0, no slot output, and B == n_supports (or
 * n_supports == 1); invalid or non-homogeneous supports are reported by
 * sfft_hidft as status 2 / 3 naming the support.  Every other entry point
 * rejects it with SFFT_ERR_INVALID. */
SFFT_API int sfft_plan_batched(const int64_t* J, int64_t k, int64_t n_supports, int M, int dtype,
                               sfft_stream_t stream, sfft_plan** plan);
SFFT_API int sfft_plan_destroy(sfft_plan* plan);
SFFT_API int sfft_plan_get_info(const sfft_plan* plan, sfft_plan_info* info);

/* Copy plan tables (bit-exact with _build_plan) to caller buffers, host or
 * device; any pointer may be NULL.  twiddles: A-1 complex of the plan dtype,
 * stage-major (stage k at offset 2^(k-1)-1).  offsets: slot order
 * (hidft.py:155-158).  Synchronises `stream`. */
SFFT_API int sfft_plan_tables(const sfft_plan* plan, int64_t* element_slots, int64_t* slot_residues,
                     uint8_t* slot_real, int64_t* node_residues, int64_t* offsets,
                     void* twiddles, sfft_stream_t stream);

/* hidft(f_b, J, r, height, shift) for B signal rows (hidft.py:135-185),
 * batched.  signals: B rows of N complex (plan dtype), row stride `ld`
 * elements.  out: B rows of n_out complex (n_out = n_nodes for NODES, k for
 * DFT/SAS, A for SLOTS), row stride ld_out.  slot_out: optional second output
 * of slot values (A per row, stride ld_slot) or NULL.
 * DFT requires a homogeneous J at height 0; SAS requires mu* = 1. */
SFFT_API int sfft_hidft(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
               int64_t shift, int out_kind, void* out, int64_t ld_out, void* slot_out,
               int64_t ld_slot, sfft_stream_t stream);

/* sfft_hidft on a batch stored sample-major: sample n of signal b at
 * signals[n * ld + b] (an (N, B) matrix, ld >= B), e.g. a device array
 * filled signal-interleaved.  The SG signals of a CTA read each needed
 * sample index as one contiguous run, so the gather moves useful sectors
 * instead of one 128 B line per sample (configs 2-4).  Outputs as
 * sfft_hidft (B rows of ld_out); 2^s <= 4096 (c64) / 2048 (c128). */
SFFT_API int sfft_hidft_interleaved(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld,
                                    int64_t shift, int out_kind, void* out, int64_t ld_out, sfft_stream_t stream);

/* Number of kernel launches sfft_hidft / sfft_hidft_gathered issue on the
 * stream for `rows` rows with this plan (1, or 2 per row chunk of the split
 * transform for 2^s beyond one CTA). */
SFFT_API int sfft_launch_count(const sfft_plan* plan, int64_t rows, int64_t* launches);

/* Programmatic dependent launch across calls, opt-in per stream.  With
 * enable = 1 the caller declares that, until the scope is closed, the
 * library's calls on `stream` are consecutive and no other kernel on the
 * stream writes their inputs: each call's first kernel may then start while
 * the previous call's last kernel drains (its loads run before
 * griddepcontrol.wait; a call whose inputs overlap an output of the chain
 * still launches fully ordered).  Default (no scope): every call's first
 * kernel is fully stream-ordered, so a foreign producer kernel that triggers
 * its dependents early can never race the library's loads.  The reference
 * has no counterpart (pure Python, no streams). */
SFFT_API int sfft_stream_chain(sfft_stream_t stream, int enable);

/* Same transform on samples already gathered in slot order (B rows of A
 * complex, row stride ld >= A): the path for callable / synthesised sources
 * (hidft.py:41-45, where the caller evaluates the signal at the offsets). */
SFFT_API int sfft_hidft_gathered(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld,
                                 int out_kind, void* out, int64_t ld_out, void* slot_out,
                                 int64_t ld_slot, sfft_stream_t stream);

/* sfft_hidft_gathered for rows in either sample order (SFFT_ORDER_PATTERN:
 * the layout sfft_host_stage writes and sfft_sas_decode's table reads). */
SFFT_API int sfft_hidft_staged(const sfft_plan* plan, const void* samples, int64_t B, int64_t ld, int order,
                               int out_kind, void* out, int64_t ld_out, void* slot_out, int64_t ld_slot,
                               sfft_stream_t stream);

/* Reorder/scale slot values (B rows, stride ld >= A) into an output kind:
 * hidft_to_dft(res) (hidft.py:188-207) or the mu*=1 SAS read (sas.py:363-371)
 * or node order. */
SFFT_API int sfft_plan_apply_map(const sfft_plan* plan, int out_kind, const void* slot_values,
                                 int64_t B, int64_t ld, void* out, int64_t ld_out,
                                 sfft_stream_t stream);

/* Measurement aid (no reference counterpart): the device's non-tensor FMA
 * throughput in the plan dtypes, from independent FMA chains on every SM
 * timed with CUDA events on `stream` (about 1 ms).  The flop side of the
 * roofline SURVEY.md 8(d) asks for; bench.py calls it in the run it reports.
 * dtype: SFFT_C64 -> fp32 FMA, SFFT_C128 -> fp64 FMA; *tflops on the host. */
SFFT_API int sfft_probe_fma_peak(int dtype, double* tflops, sfft_stream_t stream);

/* BandlimitedSignal.sample_block (core.py:164-173) on the device:
 * out[i] = (1/N) sum_e coeffs[e] exp(+2 pi i (locations[i] * J[e] mod N) / N),
 * complex128, J / coeffs / locations / out device pointers. */
SFFT_API int sfft_synthesize(const int64_t* J, const void* coeffs, int64_t k, int M,
                             const int64_t* locations, int64_t n, void* out, sfft_stream_t stream);

/* select_pivots("auto") profile (sas.py:80-113): for each prefix t = 0..s of the
 * pivot list piv (ascending pivots of J), the largest node weight mu[t] and the
 * sum of squared node weights sumsq[t] at level piv[t-1]+1 (host outputs, s+1 each). */
/* Congruence tree T^depth(J) levels level_lo..level_hi (congruence.py:134-222,
 * build_tree 217-222), built on the device.  Level l holds one node per
 * residue class mod 2^l meeting J, ascending by residue, members ascending.
 * Outputs per level i = l - level_lo: members[i*k .. i*k+k) (J permuted into
 * node order), node_off[i*(k+1) ..] (CSR: node n has members
 * node_off[n] .. node_off[n+1]-1), n_nodes[i].  Residue of node n = first
 * member mod 2^l.  Outputs may be host (synchronous) or device memory.
 * M <= 28 (one 2^M-bit rank per level). */
SFFT_API int sfft_tree_build(const int64_t* J, int64_t k, int M, int level_lo, int level_hi, int64_t* members,
                             int32_t* node_off, int32_t* n_nodes, sfft_stream_t stream);

SFFT_API int sfft_prefix_weights(const int64_t* J, int64_t k, int M, const int32_t* piv, int s,
                                 uint64_t* mu, uint64_t* sumsq, sfft_stream_t stream);

/* Node membership of a plan's decode level (congruence tree, congruence.py:134-214):
 * offsets[n_nodes+1] and member element indices (ascending J within each node),
 * host or device buffers, either may be NULL (builds and caches the table). */
SFFT_API int sfft_plan_nodes(sfft_plan* plan, int32_t* offsets, int32_t* members, sfft_stream_t stream);

/* hidft of shift0 + j for j < nshift (sas.py:343-345) in one launch: output row
 * b*nshift + j.  in_dtype may be SFFT_C64 with a complex128 plan (promoted on
 * load, as the reference's float64 path does). */
SFFT_API int sfft_hidft_shifts(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int in_dtype,
                               int64_t shift0, int64_t nshift, int out_kind, void* out, int64_t ld_out,
                               sfft_stream_t stream);

/* Shift-and-sample node decoding for mu* > 1 (sas.py:358-399): nodevals are the
 * nshift = mu* node outputs per signal (rows b*mu + j); per aliased node a
 * Bjorck-Pereyra solve with Leja order in float64, the reference's error
 * estimate, double-double re-measure/re-solve above tol/20, dense LU fallback
 * above max(tol, 1e-9) residual.  Escalation samples come from the dense
 * signals (sig), a float64 table in pattern order (table: B x mu x A), or the
 * band-limited spectra (bl_J[k_src], bl_c[B x k_src] complex128).  out: B x k
 * complex128 in ascending-J order; flags (1 escalated, 2 dense fallback) and
 * residuals per (signal, node). */
SFFT_API int sfft_sas_decode(sfft_plan* plan, const void* nodevals, int64_t ld_nv, int nv_dtype, int64_t B,
                             int64_t mu, double tol, const void* sig, int64_t ld_sig, int sig_dtype,
                             const void* table, const int64_t* bl_J, const void* bl_c, int64_t k_src,
                             const int64_t* J_dev, void* out, int64_t ld_out, int32_t* flags, double* resid,
                             int64_t* n_escalated, int64_t* n_fallback, sfft_stream_t stream);

/* Host staging gather (signals in host memory): out[b*A + a] = signals[b*ld +
 * locations[a]] for B rows of esz-byte elements (8 = complex64, 16 =
 * complex128), on a persistent pool of nthreads host threads plus the
 * caller (<= 0: all cores but the caller's).  Pure data movement feeding
 * one DMA of B*A elements; the transform then runs on the device with
 * sfft_hidft_gathered (sfft_hidft_host does both, pipelined). */
SFFT_API int sfft_host_gather(const void* signals, int64_t B, int64_t ld, int esz, const int64_t* locations,
                              int64_t A, void* out, int nthreads);

/* hidft(f_b, J, r, height, shift) for B rows resident in HOST memory
 * (pageable or page-locked), outputs to host memory: the drop-in for the
 * reference's numpy path (hidft.py:135-185, hidft_to_dft hidft.py:188-207)
 * with host arrays in and out.  Host threads gather the 2^s samples per row
 * the plan reads into page-locked staging; row chunks (chunk_rows, <= 0:
 * B/8, at least 16) are copied to the device, transformed and copied back
 * on `stream` while later chunks are still being gathered.  nthreads <= 0:
 * all cores but the caller's.  Synchronous: returns with out / slot_out
 * written.  Same output kinds and strides as sfft_hidft. */
SFFT_API int sfft_hidft_host(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int64_t shift,
                             int out_kind, void* out, int64_t ld_out, void* slot_out, int64_t ld_slot,
                             int64_t chunk_rows, int nthreads, sfft_stream_t stream);

/* Stage the samples a plan reads from HOST-resident rows into DEVICE memory:
 * output row b*nshift + j (j < nshift) holds f_b((I - shift0 - j) mod N) in
 * `order` (sfft_sample_order), A = 2^s elements per row at row stride ld_out.
 * in_dtype is the signals' type; out_dtype may be SFFT_C128 for complex64
 * signals (promoted on the host, as the reference's float64 path does,
 * sas.py:343-345).  Host threads gather while finished chunks are copied on
 * `stream`; returns once every copy is enqueued (later work on `stream` sees
 * the rows).  Feeds sfft_hidft_staged and sfft_sas_decode's sample table. */
SFFT_API int sfft_host_stage(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int in_dtype,
                             int64_t shift0, int64_t nshift, int order, int out_dtype, void* dev_out,
                             int64_t ld_out, int nthreads, sfft_stream_t stream);

/* Fused hidft(f_b, J_b, pivots(J_b)) + hidft_to_dft for homogeneous supports:
 * pivots, pattern, tables and twiddles are derived on chip per CTA, so one
 * launch does plan + gather + butterfly + scaled, ascending-J store.
 * J: n_supports rows of k indices (n_supports = 1: shared by all B signals;
 * n_supports = B: one support per signal, config 4), int64, device or host.
 * status: optional device int32[n_supports] receiving 0 / 2 / 3 per support;
 * when NULL the call synchronises and returns the worst status. */
SFFT_API int sfft_hidft_to_dft_fused(const int64_t* J, int64_t k, int64_t n_supports, int M,
                            const void* signals, int64_t B, int64_t ld, int dtype,
                            void* out, int64_t ld_out, int32_t* status,
                            sfft_stream_t stream);

/* sfft_hidft_to_dft_fused for per-signal supports (n_supports = B) with
 * signals, supports and results all in HOST memory: host threads derive each
 * support's pivots, gather its 2^s samples and stage the support, pipelined
 * with the copies; the device rebuilds each plan on chip from the support
 * and transforms the staged samples.  Synchronous; returns the worst support
 * status like the fused call with status = NULL.  k <= 2^13. */
SFFT_API int sfft_hidft_to_dft_fused_host(const int64_t* J, int64_t k, int M, const void* signals, int64_t B,
                                          int64_t ld, int dtype, void* out, int64_t ld_out, int nthreads,
                                          sfft_stream_t stream);

/* ---- result rows in another process's device memory ----
 * The reference returns each signal's coefficients to its caller
 * (hidft.py:188-207); with the batch sharded over the GPUs of a node the
 * rows end up on one rank.  The owner allocates the B x k result buffer and
 * exports a CUDA IPC handle (SFFT_IPC_HANDLE_BYTES opaque bytes, sent to the
 * other ranks by the caller); each other rank maps it and passes its row
 * shard of the mapped pointer as the `out` of sfft_hidft /
 * sfft_hidft_to_dft_fused, so the transform's own stores write the rows
 * over NVLink / NVSwitch peer memory (no separate gather collective).  The
 * writer synchronises its stream before the owner reads (e.g. a barrier). */
#define SFFT_IPC_HANDLE_BYTES 64
SFFT_API int sfft_peer_alloc(int64_t bytes, void** dptr, unsigned char* handle);
SFFT_API int sfft_peer_free(void* dptr);
SFFT_API int sfft_peer_open(const unsigned char* handle, void** dptr);
SFFT_API int sfft_peer_close(void* dptr);

#ifdef __cplusplus
}
#endif
#endif /* STRUCTFFT_B200_H */
