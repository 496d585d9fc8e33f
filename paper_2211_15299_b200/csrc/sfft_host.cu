// Host-resident signals.  Only the 2^s samples per row that the transform
// reads ever cross PCIe: a persistent pool of host threads gathers them
// (plan offsets, slot order) into page-locked staging, and the calling thread
// streams finished row chunks to the device (DMA), runs the gathered
// transform (sfft_hidft_gathered) and copies each chunk's result back, so
// gather, both DMA directions and the kernel overlap chunk by chunk.  Rows
// are handed out through an atomic counter (no static partition: a
// descheduled worker does not stall a chunk) and the calling thread gathers
// too while it has nothing to enqueue.  Pure data movement on the host.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "sfft_common.cuh"
#include "sfft_plan.h"

namespace sfft {

class HostPool {
 public:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  int size() const { return (int)workers_.size(); }
  // start fn(worker) on every worker; returns at once
  void start(const std::function<void(int)>* fn) {
    std::lock_guard<std::mutex> lk(mu_);
    job_ = fn;
    pending_ = (int)workers_.size();
    ++gen_;
    cv_.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(i);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

static std::mutex g_host_mu;  // one host job at a time through the shared pool and staging

// SFFT_HOST_TRACE=1: per-call timeline of the host pipeline on stderr (probe only)
static bool host_trace() {
  static const bool v = [] { const char* e = getenv("SFFT_HOST_TRACE"); return e && atoi(e) != 0; }();
  return v;
}
static double now_us() {
  using namespace std::chrono;
  return duration<double, std::micro>(steady_clock::now().time_since_epoch()).count();
}
static HostPool* g_pool = nullptr;

// default: every core but the calling thread's (which gathers too), shared
// between the processes of one node under torchrun (LOCAL_WORLD_SIZE)
static int default_threads() {
  if (const char* e = getenv("SFFT_HOST_THREADS"))  // explicit pool size (probes)
    if (atoi(e) > 0) return atoi(e);
  int hw = (int)std::thread::hardware_concurrency();
  if (const char* e = getenv("LOCAL_WORLD_SIZE")) hw /= std::max(1, atoi(e));
  return std::max(1, hw - 1);
}

static HostPool& pool(int want) {  // caller holds g_host_mu
  const int n = want > 0 ? want : default_threads();
  if (!g_pool || g_pool->size() != n) {
    delete g_pool;
    g_pool = new HostPool(n);
  }
  return *g_pool;
}

// below this many samples a job runs on the calling thread alone
constexpr int64_t kPoolMinSamples = 1 << 13;

struct C64b { uint64_t v; };
struct C128b { uint64_t lo, hi; };

template <typename In, typename Out> struct Elem {
  static Out conv(In v) { return v; }
};
template <> struct Elem<float2, double2> {
  static double2 conv(float2 v) { return {(double)v.x, (double)v.y}; }
};

// Row dispenser shared by the pool and the calling thread.  Unit = one
// source row, which produces nshift output rows: row j holds
// src[(loc[a] - j) & nmask] for a < A (the shifts of one sample share its
// cache line, so a row is read once for all of them).
struct RowJob {
  const char* sig = nullptr;
  int64_t ld_bytes = 0, B = 0, A = 0, nshift = 1, grain = 1, chunk = 1;
  uint64_t nmask = ~0ull;
  int in_esz = 8, out_esz = 8;
  const int64_t* loc = nullptr;
  // runs of consecutive locations (pattern order with the top pivots at the
  // top bits of the index, config 5: 16-sample runs = 128 B lines): copied
  // as blocks instead of sample by sample
  std::vector<std::pair<int64_t, int64_t>> runs;  // (first index a, length)
  char* out = nullptr;
  std::atomic<int64_t> next{0};
  std::unique_ptr<std::atomic<int64_t>[]> done;  // source rows finished per chunk
  const std::function<void(int64_t)>* row_fn = nullptr;  // custom per-row work (replaces the gather)

  template <typename In, typename Out>
  void rows(int64_t r0, int64_t r1) const {
    for (int64_t r = r0; r < r1; ++r) {
      const In* row = reinterpret_cast<const In*>(sig + r * ld_bytes);
      Out* o = reinterpret_cast<Out*>(out) + r * nshift * A;
      if (nshift == 1 && nmask == ~0ull && !runs.empty() && sizeof(In) == sizeof(Out)) {
        for (const auto& ru : runs) std::memcpy(o + ru.first, row + loc[ru.first], (size_t)ru.second * sizeof(In));
      } else if (nshift == 1 && nmask == ~0ull) {
        for (int64_t a = 0; a < A; ++a) o[a] = Elem<In, Out>::conv(row[loc[a]]);
      } else {
        for (int64_t a = 0; a < A; ++a) {
          const uint64_t p = (uint64_t)loc[a];
          for (int64_t j = 0; j < nshift; ++j) o[j * A + a] = Elem<In, Out>::conv(row[(p - (uint64_t)j) & nmask]);
        }
      }
    }
  }
  // gather one grain of source rows; false when none is left
  bool step() {
    const int64_t r0 = next.fetch_add(grain, std::memory_order_relaxed);
    if (r0 >= B) return false;
    const int64_t r1 = std::min(B, r0 + grain);
    if (row_fn) for (int64_t r = r0; r < r1; ++r) (*row_fn)(r);
    else if (in_esz == 8 && out_esz == 8) rows<C64b, C64b>(r0, r1);
    else if (in_esz == 8) rows<float2, double2>(r0, r1);
    else rows<C128b, C128b>(r0, r1);
    // grains never straddle chunks (chunk is a multiple of grain)
    if (done) done[r0 / chunk].fetch_add(r1 - r0, std::memory_order_release);
    return true;
  }
  // block copies when the locations form runs of >= 4 samples on average
  void find_runs() {
    runs.clear();
    if (!loc || A == 0 || nshift != 1 || nmask != ~0ull) return;
    for (int64_t a = 0; a < A;) {
      int64_t e = a + 1;
      while (e < A && loc[e] == loc[e - 1] + 1) ++e;
      runs.emplace_back(a, e - a);
      a = e;
    }
    if ((int64_t)runs.size() * 4 > A) runs.clear();
  }
  void set_chunking(int64_t chunk_rows) {
    grain = std::max<int64_t>(1, 4096 / std::max<int64_t>(A * nshift, 1));
    // default B/16, at least 32 rows (config 2: 128 / 64 / 32 / 16 / 8 rows -> 1.13 / 1.09 / 1.10 / 1.5 / 2.1 ms)
    int64_t c = chunk_rows > 0 ? chunk_rows : std::max<int64_t>(32, (B + 15) / 16);
    chunk = (c + grain - 1) / grain * grain;
    const int64_t n = (B + chunk - 1) / chunk;
    done.reset(new std::atomic<int64_t>[n]);
    for (int64_t k = 0; k < n; ++k) done[k].store(0, std::memory_order_relaxed);
  }
  int64_t nchunks() const { return (B + chunk - 1) / chunk; }
  int64_t chunk_rows(int64_t c) const { return std::min(chunk, B - c * chunk); }
  // calling thread: wait for chunk c, gathering rows itself meanwhile
  void await(int64_t c) {
    const int64_t want = chunk_rows(c);
    while (done[c].load(std::memory_order_acquire) < want)
      if (!step()) std::this_thread::yield();
  }
};

// Page-locked and device staging, grown on demand, reused across calls
// (page-locking per call costs more than the transfer).  h_free is recorded
// after the last copy that reads h_in; the next job waits on it before
// overwriting the staging.
struct Staging {
  void* h_in = nullptr;  size_t h_in_n = 0;
  void* h_out = nullptr; size_t h_out_n = 0;
  void* d_in = nullptr;  size_t d_in_n = 0;
  void* d_out = nullptr; size_t d_out_n = 0;
  void* d_slot = nullptr; size_t d_slot_n = 0;
  void* h_J = nullptr;   size_t h_J_n = 0;   // per-signal supports (fused host path)
  void* d_J = nullptr;   size_t d_J_n = 0;
  void* d_stat = nullptr; size_t d_stat_n = 0;
  cudaEvent_t h_free = nullptr;
  // device->host copies run on their own stream so chunk c's result copy
  // overlaps chunk c+1's host->device copy (the two DMA directions); the
  // caller's stream waits for it before the call returns
  cudaStream_t d2h = nullptr;
  cudaEvent_t ev_k = nullptr, ev_d2h = nullptr;
  int device = -1;
};
static Staging g_stage;

static int grow_host(void** p, size_t* n, size_t want) {
  if (*n >= want) return SFFT_OK;
  if (*p) cudaFreeHost(*p);
  *p = nullptr;
  *n = 0;
  SFFT_CUDA(cudaHostAlloc(p, want, cudaHostAllocPortable));
  *n = want;
  return SFFT_OK;
}
static int grow_dev(void** p, size_t* n, size_t want) {
  if (*n >= want) return SFFT_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *n = 0;
  SFFT_CUDA(cudaMalloc(p, want));
  *n = want;
  return SFFT_OK;
}

// caller holds g_host_mu: staging of the current device, h_in free to write
static int stage_begin(int dev) {
  Staging& S = g_stage;
  if (S.h_free) SFFT_CUDA(cudaEventSynchronize(S.h_free));
  if (S.device != dev) {  // device buffers of another device: drop them
    if (S.d_in) cudaFree(S.d_in);
    if (S.d_out) cudaFree(S.d_out);
    if (S.d_slot) cudaFree(S.d_slot);
    if (S.d_J) cudaFree(S.d_J);
    if (S.d_stat) cudaFree(S.d_stat);
    if (S.h_free) cudaEventDestroy(S.h_free);
    if (S.d2h) cudaStreamDestroy(S.d2h);
    if (S.ev_k) cudaEventDestroy(S.ev_k);
    if (S.ev_d2h) cudaEventDestroy(S.ev_d2h);
    S.d_in = S.d_out = S.d_slot = S.d_J = S.d_stat = nullptr;
    S.d_in_n = S.d_out_n = S.d_slot_n = S.d_J_n = S.d_stat_n = 0;
    S.h_free = nullptr;
    S.d2h = nullptr;
    S.ev_k = S.ev_d2h = nullptr;
    S.device = dev;
  }
  if (!S.h_free) SFFT_CUDA(cudaEventCreateWithFlags(&S.h_free, cudaEventDisableTiming));
  if (!S.ev_k) SFFT_CUDA(cudaEventCreateWithFlags(&S.ev_k, cudaEventDisableTiming));
  if (!S.ev_d2h) SFFT_CUDA(cudaEventCreateWithFlags(&S.ev_d2h, cudaEventDisableTiming));
  if (!S.d2h) SFFT_CUDA(cudaStreamCreateWithFlags(&S.d2h, cudaStreamNonBlocking));
  return SFFT_OK;
}

// the result copies of the chunk just enqueued on st go to the D2H stream
static cudaError_t d2h_after(cudaStream_t st) {
  cudaError_t e = cudaEventRecord(g_stage.ev_k, st);
  return e == cudaSuccess ? cudaStreamWaitEvent(g_stage.d2h, g_stage.ev_k, 0) : e;
}
// the caller's stream waits for every result copy
static cudaError_t d2h_join(cudaStream_t st) {
  cudaError_t e = cudaEventRecord(g_stage.ev_d2h, g_stage.d2h);
  return e == cudaSuccess ? cudaStreamWaitEvent(st, g_stage.ev_d2h, 0) : e;
}

static bool is_pinned_host(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// sample locations of a plan, shift0 applied: slot order (hidft.py:155-158)
// or ascending pattern order (pattern position u holds slot brev_s(u))
static std::vector<int64_t> plan_locations(const sfft_plan* p, int64_t shift0, bool pattern_order) {
  const int64_t N = 1ll << p->M, A = p->A;
  const int64_t sh = ((shift0 % N) + N) % N;
  // loc[u] = loc[u without its lowest set bit] + that bit's stride: O(A)
  // (the per-bit sum was ~1 ms per call at A = 2^16)
  int64_t d[64];
  for (int j = 0; j < p->s; ++j) {
    const int i = pattern_order ? p->s - 1 - j : j;  // index bit j <-> slot bit i
    d[j] = 1ll << (p->M - 1 - p->used[i]);
  }
  std::vector<int64_t> loc(A);
  if (A > 0) loc[0] = 0;
  for (int64_t u = 1; u < A; ++u) loc[u] = loc[u & (u - 1)] + d[__builtin_ctzll((unsigned long long)u)];
  for (int64_t u = 0; u < A; ++u) loc[u] = (loc[u] - sh + N) & (N - 1);
  return loc;
}

}  // namespace sfft

using namespace sfft;

extern "C" int sfft_host_gather(const void* signals, int64_t B, int64_t ld, int esz, const int64_t* locations,
                                int64_t A, void* out, int nthreads) {
  SFFT_NVTX("sfft_host_gather");
  if (!signals || !locations || !out) return fail(SFFT_ERR_INVALID, "null pointer");
  if (esz != 8 && esz != 16) return fail(SFFT_ERR_INVALID, "element size must be 8 or 16 bytes");
  if (B < 0 || A < 0 || ld < 0) return fail(SFFT_ERR_INVALID, "negative size");
  if (B == 0 || A == 0) return SFFT_OK;
  std::lock_guard<std::mutex> lk(g_host_mu);
  HostPool& p = pool(nthreads);
  RowJob job;
  job.sig = (const char*)signals;
  job.ld_bytes = ld * esz;
  job.B = B;
  job.A = A;
  job.in_esz = job.out_esz = esz;
  job.loc = locations;
  job.out = (char*)out;
  job.grain = std::max<int64_t>(1, 4096 / A);
  const std::function<void(int)> fn = [&job](int) { while (job.step()) {} };
  p.start(&fn);
  while (job.step()) {}
  p.wait();
  return SFFT_OK;
}

extern "C" int sfft_hidft_host(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int64_t shift,
                               int out_kind, void* out, int64_t ld_out, void* slot_out, int64_t ld_slot,
                               int64_t chunk_rows, int nthreads, sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_host");
  cudaStream_t st = (cudaStream_t)stream;
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(plan, "sfft_hidft_host")) return rj;
  if (B < 0) return fail(SFFT_ERR_INVALID, "negative batch");
  const int32_t* map = nullptr;
  int64_t n_out = 0;
  double scale = 1.0;
  int rc = out_spec(plan, out_kind, &map, &n_out, &scale);
  if (rc) return rc;
  if (B == 0) return SFFT_OK;
  if (!signals || !out) return fail(SFFT_ERR_INVALID, "null signal or output pointer");
  const int64_t N = 1ll << plan->M, A = plan->A;
  if (ld < N) return fail(SFFT_ERR_INVALID, "signal row stride too small");
  if (ld_out < n_out) return fail(SFFT_ERR_INVALID, "output row stride too small");
  if (slot_out && ld_slot < A) return fail(SFFT_ERR_INVALID, "slot row stride too small");
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  if (dev != plan->device) return fail(SFFT_ERR_INVALID, "plan belongs to another device");
  const int esz = plan->dtype == SFFT_C64 ? 8 : 16;
  // the cluster transform reads pre-gathered rows in pattern order: stage
  // them that way there (coalesced on the device, ascending on the host)
  const bool sorted = gathered_sorted(plan);
  const double t_call = host_trace() ? now_us() : 0.0;
  const std::vector<int64_t> loc = plan_locations(plan, shift, sorted);

  std::lock_guard<std::mutex> lk(g_host_mu);
  if ((rc = stage_begin(dev))) return rc;
  Staging& S = g_stage;
  const bool out_pinned = is_pinned_host(out);
  const bool slot_pinned = !slot_out || is_pinned_host(slot_out);
  const size_t in_bytes = (size_t)B * A * esz, out_bytes = (size_t)B * n_out * esz;
  const size_t slot_bytes = slot_out ? (size_t)B * A * esz : 0;
  if ((rc = grow_host(&S.h_in, &S.h_in_n, in_bytes))) return rc;
  if ((rc = grow_dev(&S.d_in, &S.d_in_n, in_bytes))) return rc;
  if ((rc = grow_dev(&S.d_out, &S.d_out_n, out_bytes))) return rc;
  if (slot_out && (rc = grow_dev(&S.d_slot, &S.d_slot_n, slot_bytes))) return rc;
  if ((!out_pinned || !slot_pinned) &&
      (rc = grow_host(&S.h_out, &S.h_out_n, (out_pinned ? 0 : out_bytes) + (slot_pinned ? 0 : slot_bytes))))
    return rc;
  char* out_tgt = out_pinned ? (char*)out : (char*)S.h_out;
  const int64_t ldo_tgt = out_pinned ? ld_out : n_out;
  char* slot_tgt = slot_out ? (slot_pinned ? (char*)slot_out : (char*)S.h_out + (out_pinned ? 0 : out_bytes)) : nullptr;
  const int64_t lds_tgt = slot_pinned ? ld_slot : A;

  // Optionally (SFFT_HOST_GPU_FRACTION) the device reads the first g0
  // page-locked rows itself, zero-copy over PCIe, while the host threads
  // gather the rest.  Measured on config 2 (tools/e2e_probe.py): 0.1 / 0.2 /
  // 0.3 of the rows -> 1.31 / 1.52 / 1.87 ms against 1.1 ms host-only (the
  // per-sample PCIe reads are slow and compete for host memory), so 0.
  static const double gpu_frac = [] {
    const char* e = getenv("SFFT_HOST_GPU_FRACTION");
    return e ? std::min(1.0, std::max(0.0, atof(e))) : 0.0;
  }();
  const int64_t g0 = is_pinned_host(signals) ? (int64_t)(gpu_frac * (double)B) : 0;
  if (g0 > 0) {
    rc = sfft_hidft(plan, signals, g0, ld, shift, out_kind, S.d_out, n_out, slot_out ? S.d_slot : nullptr, A,
                    stream);
    cudaError_t e = rc ? cudaSuccess
                       : cudaMemcpy2DAsync(out_tgt, (size_t)ldo_tgt * esz, S.d_out, (size_t)n_out * esz,
                                           (size_t)n_out * esz, g0, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && !rc && slot_out)
      e = cudaMemcpy2DAsync(slot_tgt, (size_t)lds_tgt * esz, S.d_slot, (size_t)A * esz, (size_t)A * esz, g0,
                            cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "device->host copy");
    if (rc) return rc;
  }

  RowJob job;
  job.sig = (const char*)signals + (size_t)g0 * ld * esz;
  job.ld_bytes = ld * esz;
  job.B = B - g0;
  job.A = A;
  job.in_esz = job.out_esz = esz;
  job.loc = loc.data();
  job.out = (char*)S.h_in;
  job.find_runs();
  job.set_chunking(chunk_rows);

  // small jobs: the calling thread alone (waking the pool costs more)
  const bool use_pool = job.B > 0 && job.B * A >= kPoolMinSamples;
  HostPool& p = pool(nthreads);
  const std::function<void(int)> fn = [&job](int) { while (job.step()) {} };
  if (use_pool) p.start(&fn);
  const bool tr = host_trace();
  const double t0 = tr ? now_us() : 0.0;
  std::vector<double> tw;
  std::vector<cudaEvent_t> tev;  // per chunk: before H2D, after H2D, after transform, after D2H
  for (int64_t c = 0; c < job.nchunks() && job.B > 0 && rc == SFFT_OK; ++c) {
    job.await(c);
    if (tr) tw.push_back(now_us() - t0);
    const int64_t rows = job.chunk_rows(c);
    const int64_t hb = c * job.chunk, b0 = g0 + hb;  // row in the staging / in the batch
    const size_t ib = (size_t)hb * A * esz;
    char* din = (char*)S.d_in + ib;
    char* dout = (char*)S.d_out + (size_t)b0 * n_out * esz;
    char* dslot = slot_out ? (char*)S.d_slot + (size_t)b0 * A * esz : nullptr;
    if (tr) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), st); }
    cudaError_t e = cudaMemcpyAsync(din, (char*)S.h_in + ib, (size_t)rows * A * esz, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "host->device chunk copy"); break; }
    if (tr) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), st); }
    rc = hidft_gathered(plan, din, rows, A, sorted, out_kind, dout, n_out, dslot, A, st);
    if (rc) break;
    if (tr) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), st); }
    e = d2h_after(st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(out_tgt + (size_t)b0 * ldo_tgt * esz, (size_t)ldo_tgt * esz, dout, (size_t)n_out * esz,
                            (size_t)n_out * esz, rows, cudaMemcpyDeviceToHost, S.d2h);
    if (e == cudaSuccess && slot_out)
      e = cudaMemcpy2DAsync(slot_tgt + (size_t)b0 * lds_tgt * esz, (size_t)lds_tgt * esz, dslot, (size_t)A * esz,
                            (size_t)A * esz, rows, cudaMemcpyDeviceToHost, S.d2h);
    if (tr) { tev.emplace_back(); cudaEventCreate(&tev.back()); cudaEventRecord(tev.back(), S.d2h); }
    if (e != cudaSuccess) rc = cuda_fail(e, "device->host chunk copy");
  }
  const cudaError_t ej = d2h_join(st);
  if (ej != cudaSuccess && rc == SFFT_OK) rc = cuda_fail(ej, "device->host stream join");
  if (use_pool) {
    while (job.step()) {}  // on error: drain so no worker still reads the caller's rows
    p.wait();
  }
  const double t_enq = tr ? now_us() - t0 : 0.0;
  cudaEventRecord(S.h_free, st);
  const cudaError_t es = cudaStreamSynchronize(st);
  if (tr) {
    fprintf(stderr, "[sfft host] B=%lld A=%lld chunks=%lld chunk=%lld pool=%d out_pinned=%d: setup %.0f us, await(c) us:",
            (long long)B, (long long)A, (long long)job.nchunks(), (long long)job.chunk, (int)use_pool,
            (int)out_pinned, t0 - t_call);
    for (double x : tw) fprintf(stderr, " %.0f", x);
    fprintf(stderr, " | enqueued %.0f | synced %.0f\n", t_enq, now_us() - t0);
    for (size_t i = 0; i + 3 < tev.size(); i += 4) {
      float h2d = 0, k = 0, d2h = 0, from0 = 0;
      cudaEventElapsedTime(&h2d, tev[i], tev[i + 1]);
      cudaEventElapsedTime(&k, tev[i + 1], tev[i + 2]);
      cudaEventElapsedTime(&d2h, tev[i + 2], tev[i + 3]);
      cudaEventElapsedTime(&from0, tev[0], tev[i + 3]);
      fprintf(stderr, "[sfft host]   chunk %zu: h2d %.0f us, transform %.0f us, d2h %.0f us, done at %.0f us\n", i / 4,
              h2d * 1e3, k * 1e3, d2h * 1e3, from0 * 1e3);
    }
    for (cudaEvent_t ev : tev) cudaEventDestroy(ev);
  }
  if (rc) return rc;
  if (es != cudaSuccess) return cuda_fail(es, "host transform");
  // pageable outputs: copy out of the pinned result staging
  for (int k = 0; k < 2; ++k) {
    const bool slot = k == 1;
    if (slot ? (!slot_out || slot_pinned) : out_pinned) continue;
    const char* src = slot ? slot_tgt : out_tgt;
    char* dst = (char*)(slot ? slot_out : out);
    const int64_t w = slot ? A : n_out, ldd = slot ? ld_slot : ld_out;
    for (int64_t b = 0; b < B; ++b) std::memcpy(dst + (size_t)b * ldd * esz, src + (size_t)b * w * esz, (size_t)w * esz);
  }
  return SFFT_OK;
}

extern "C" int sfft_host_stage(const sfft_plan* plan, const void* signals, int64_t B, int64_t ld, int in_dtype,
                               int64_t shift0, int64_t nshift, int order, int out_dtype, void* dev_out,
                               int64_t ld_out, int nthreads, sfft_stream_t stream) {
  SFFT_NVTX("sfft_host_stage");
  cudaStream_t st = (cudaStream_t)stream;
  if (!plan) return fail(SFFT_ERR_INVALID, "null plan");
  if (int rj = reject_per_signal(plan, "sfft_host_stage")) return rj;
  if (B < 0 || nshift < 1) return fail(SFFT_ERR_INVALID, "negative batch or nshift < 1");
  if (in_dtype != SFFT_C64 && in_dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown input dtype");
  if (out_dtype != SFFT_C64 && out_dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown output dtype");
  if (in_dtype == SFFT_C128 && out_dtype == SFFT_C64)
    return fail(SFFT_ERR_INVALID, "complex128 signals cannot be staged as complex64");
  if (order != SFFT_ORDER_SLOT && order != SFFT_ORDER_PATTERN) return fail(SFFT_ERR_INVALID, "unknown sample order");
  if (B == 0) return SFFT_OK;
  if (!signals || !dev_out) return fail(SFFT_ERR_INVALID, "null signal or output pointer");
  const int64_t N = 1ll << plan->M, A = plan->A;
  if (ld < N) return fail(SFFT_ERR_INVALID, "signal row stride too small");
  if (ld_out < A) return fail(SFFT_ERR_INVALID, "output row stride too small");
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));
  if (dev != plan->device) return fail(SFFT_ERR_INVALID, "plan belongs to another device");
  const int iesz = in_dtype == SFFT_C64 ? 8 : 16, oesz = out_dtype == SFFT_C64 ? 8 : 16;
  const std::vector<int64_t> loc = plan_locations(plan, shift0, order == SFFT_ORDER_PATTERN);

  std::lock_guard<std::mutex> lk(g_host_mu);
  int rc = stage_begin(dev);
  if (rc) return rc;
  Staging& S = g_stage;
  const int64_t rowlen = nshift * A;  // output elements per source row
  if ((rc = grow_host(&S.h_in, &S.h_in_n, (size_t)B * rowlen * oesz))) return rc;
  RowJob job;
  job.sig = (const char*)signals;
  job.ld_bytes = ld * iesz;
  job.B = B;
  job.A = A;
  job.nshift = nshift;
  job.nmask = (uint64_t)(N - 1);
  job.in_esz = iesz;
  job.out_esz = oesz;
  job.loc = loc.data();
  job.out = (char*)S.h_in;
  job.set_chunking(0);

  const bool use_pool = B * rowlen >= kPoolMinSamples;
  HostPool& p = pool(nthreads);
  const std::function<void(int)> fn = [&job](int) { while (job.step()) {} };
  if (use_pool) p.start(&fn);
  for (int64_t c = 0; c < job.nchunks() && rc == SFFT_OK; ++c) {
    job.await(c);
    const int64_t r0 = c * job.chunk * nshift, rows = job.chunk_rows(c) * nshift;  // output rows
    const cudaError_t e = cudaMemcpy2DAsync((char*)dev_out + (size_t)r0 * ld_out * oesz, (size_t)ld_out * oesz,
                                            (char*)S.h_in + (size_t)r0 * A * oesz, (size_t)A * oesz,
                                            (size_t)A * oesz, rows, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "host->device staging copy");
  }
  if (use_pool) {
    while (job.step()) {}
    p.wait();
  }
  cudaEventRecord(S.h_free, st);
  return rc;
}

// hidft_to_dft for per-signal supports with signals, supports and results in
// HOST memory (config 4 from numpy): per row the host threads derive the
// support's pivots (homogeneous: the set bits of OR_j 2^v2(j ^ j_0)), gather
// the 2^s samples in slot order and stage the support; chunks of rows go to
// the device, where the fused kernel rebuilds each plan on chip from the
// support and transforms the staged samples.  Invalid supports are staged as
// zeros and reported by the device as status 2 / 3 naming the support.
extern "C" int sfft_hidft_to_dft_fused_host(const int64_t* J, int64_t k, int M, const void* signals, int64_t B,
                                            int64_t ld, int dtype, void* out, int64_t ld_out, int nthreads,
                                            sfft_stream_t stream) {
  SFFT_NVTX("sfft_hidft_to_dft_fused_host");
  cudaStream_t st = (cudaStream_t)stream;
  if (M < 1 || M > 31) return fail(SFFT_ERR_INVALID, "M must lie in [1, 31]");
  if (dtype != SFFT_C64 && dtype != SFFT_C128) return fail(SFFT_ERR_INVALID, "unknown dtype");
  if (k < 1) return fail(SFFT_ERR_INVALID, "support set is empty");
  if (B < 0) return fail(SFFT_ERR_INVALID, "negative batch");
  if (B == 0) return SFFT_OK;
  if (!J || !signals || !out) return fail(SFFT_ERR_INVALID, "null pointer");
  if (is_device_pointer(J) && !is_pinned_host(J)) return fail(SFFT_ERR_INVALID, "supports must be in host memory");
  const int64_t N = 1ll << M;
  if (ld < N) return fail(SFFT_ERR_INVALID, "signal row stride smaller than N");
  if (ld_out < k) return fail(SFFT_ERR_INVALID, "output row stride too small");
  if (k & (k - 1)) return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support");
  const int s = 63 - __builtin_clzll((unsigned long long)k);
  const int64_t A = k;
  const int esz = dtype == SFFT_C64 ? 8 : 16;
  int dev = 0;
  SFFT_CUDA(cudaGetDevice(&dev));

  std::lock_guard<std::mutex> lk(g_host_mu);
  int rc = stage_begin(dev);
  if (rc) return rc;
  Staging& Sg = g_stage;
  const bool out_pinned = is_pinned_host(out);
  const size_t in_bytes = (size_t)B * A * esz, out_bytes = (size_t)B * k * esz, j_bytes = (size_t)B * k * 8;
  if ((rc = grow_host(&Sg.h_in, &Sg.h_in_n, in_bytes))) return rc;
  if ((rc = grow_host(&Sg.h_J, &Sg.h_J_n, j_bytes))) return rc;
  if ((rc = grow_dev(&Sg.d_in, &Sg.d_in_n, in_bytes))) return rc;
  if ((rc = grow_dev(&Sg.d_out, &Sg.d_out_n, out_bytes))) return rc;
  if ((rc = grow_dev(&Sg.d_J, &Sg.d_J_n, j_bytes))) return rc;
  if ((rc = grow_dev(&Sg.d_stat, &Sg.d_stat_n, (size_t)B * 4))) return rc;
  if (!out_pinned && (rc = grow_host(&Sg.h_out, &Sg.h_out_n, out_bytes))) return rc;
  char* out_tgt = out_pinned ? (char*)out : (char*)Sg.h_out;
  const int64_t ldo_tgt = out_pinned ? ld_out : k;

  const char* sig = (const char*)signals;
  char* h_in = (char*)Sg.h_in;
  int64_t* h_J = (int64_t*)Sg.h_J;
  const std::function<void(int64_t)> row_fn = [&](int64_t r) {
    const int64_t* Jr = J + r * k;
    std::memcpy(h_J + r * k, Jr, (size_t)k * 8);
    char* o = h_in + (size_t)r * A * esz;
    // pivots of a homogeneous support (congruence.py:76-101): the levels v2(j - j_0)
    bool ok = Jr[0] >= 0 && Jr[0] < N;
    uint64_t mask = 0;
    for (int64_t e = 1; e < k && ok; ++e) {
      ok = Jr[e] > Jr[e - 1] && Jr[e] < N;
      if (!ok) break;  // strictly increasing: Jr[e] != Jr[0], so the ctz below is defined
      mask |= 1ull << __builtin_ctzll((unsigned long long)(Jr[e] ^ Jr[0]));
    }
    if (!ok || __builtin_popcountll(mask) != s) {  // the device reports it
      std::memset(o, 0, (size_t)A * esz);
      return;
    }
    int64_t d[32];
    for (int i = 0; i < s; ++i) {
      const int piv = __builtin_ctzll(mask);
      mask &= mask - 1;
      d[i] = 1ll << (M - 1 - piv);  // hidft.py:155-158
    }
    const char* row = sig + (size_t)r * ld * esz;
    int64_t offs[1 << 13];
    offs[0] = 0;
    for (int64_t a = 1; a < A; ++a) offs[a] = offs[a & (a - 1)] + d[__builtin_ctzll((unsigned long long)a)];
    if (esz == 8) {
      const C64b* rw = (const C64b*)row;
      C64b* ow = (C64b*)o;
      for (int64_t a = 0; a < A; ++a) ow[a] = rw[offs[a]];
    } else {
      const C128b* rw = (const C128b*)row;
      C128b* ow = (C128b*)o;
      for (int64_t a = 0; a < A; ++a) ow[a] = rw[offs[a]];
    }
  };
  if (A > (1 << 13)) return fail(SFFT_ERR_UNSUPPORTED, "host fused path limited to 2^13 slots");

  RowJob job;
  job.B = B;
  job.A = A;
  job.row_fn = &row_fn;
  job.set_chunking(0);
  const bool use_pool = B * A >= kPoolMinSamples;
  HostPool& p = pool(nthreads);
  const std::function<void(int)> fn = [&job](int) { while (job.step()) {} };
  if (use_pool) p.start(&fn);
  int32_t* dstat = (int32_t*)Sg.d_stat;
  for (int64_t c = 0; c < job.nchunks() && rc == SFFT_OK; ++c) {
    job.await(c);
    const int64_t b0 = c * job.chunk, rows = job.chunk_rows(c);
    char* din = (char*)Sg.d_in + (size_t)b0 * A * esz;
    int64_t* dJ = (int64_t*)Sg.d_J + b0 * k;
    char* dout = (char*)Sg.d_out + (size_t)b0 * k * esz;
    cudaError_t e = cudaMemcpyAsync(din, h_in + (size_t)b0 * A * esz, (size_t)rows * A * esz,
                                    cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dJ, h_J + b0 * k, (size_t)rows * k * 8, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { rc = cuda_fail(e, "host->device chunk copy"); break; }
    rc = fused_to_dft(dJ, k, rows, M, din, rows, A, dtype, dout, k, dstat + b0, st, 1);
    if (rc) break;
    e = d2h_after(st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(out_tgt + (size_t)b0 * ldo_tgt * esz, (size_t)ldo_tgt * esz, dout, (size_t)k * esz,
                            (size_t)k * esz, rows, cudaMemcpyDeviceToHost, Sg.d2h);
    if (e != cudaSuccess) rc = cuda_fail(e, "device->host chunk copy");
  }
  const cudaError_t ej = d2h_join(st);
  if (ej != cudaSuccess && rc == SFFT_OK) rc = cuda_fail(ej, "device->host stream join");
  if (use_pool) {
    while (job.step()) {}
    p.wait();
  }
  std::vector<int32_t> hs((size_t)B);
  cudaEventRecord(Sg.h_free, st);
  cudaError_t es = rc ? cudaSuccess : cudaMemcpyAsync(hs.data(), dstat, (size_t)B * 4, cudaMemcpyDeviceToHost, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (rc) return rc;
  if (es != cudaSuccess || e2 != cudaSuccess) return cuda_fail(es != cudaSuccess ? es : e2, "fused host transform");
  for (int64_t i = 0; i < B; ++i) {
    if (hs[i] == 2) return fail(SFFT_ERR_INVALID, "support " + std::to_string(i) + " is not a valid SupportSet");
    if (hs[i] == 3)
      return fail(SFFT_ERR_CONTRACT, "hidft_to_dft requires a homogeneous support (support " + std::to_string(i) + ")");
  }
  if (!out_pinned)
    for (int64_t b = 0; b < B; ++b)
      std::memcpy((char*)out + (size_t)b * ld_out * esz, out_tgt + (size_t)b * k * esz, (size_t)k * esz);
  return SFFT_OK;
}
