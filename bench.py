#!/usr/bin/env python3
"""Throughput bench of the B200 Hi-DFT (BASELINE.json metric: support-DFT
coeffs/s = B*k/s, and the fraction of the HBM-gather roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A step is one pass of the hot path -- hidft(f_b, J, pivots(J)) +
hidft_to_dft for every signal of the batch -- over one batch of synthetic
signals resident in HBM.  The headline workload is BASELINE config 2
(N=2^20, k=1024, B=1024 signals per GPU sharing one support, complex64); at
N=1 the same run also measures configs 1, 3, 4, 5 and 5's complex128 pass
(`per_config`).  --gpus N > 1 without torchrun re-launches this script under
torch.distributed.run with N ranks (127.0.0.1); each rank owns its own
batch (weak scaling, no data-path collective; --scaling strong shards the
config's batch), the timed region is bracketed by a barrier and a device
synchronise and the max over ranks is reported.

L2: the gather footprint of one batch (~32-40 MiB) fits in the 126 MB L2,
so the timed steps rotate over R input sets whose combined footprint is
several times L2 (each set is the same signals at different addresses).

--impl reference times the UNMODIFIED reference package (structfft,
installed into baseline/_ref by `pip install --target baseline/_ref`) on
the host cores with a process pool, on a bounded sample of the same
workload; without that install it falls back to the numpy port in oracle/
(kind "port", pinned to the reference by golden vectors).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "support-DFT coeffs/s (B·k/s)"
UNIT = "coeffs/s"


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ------------------------------------------------------------- clocks ---

class ClockSampler:
    """nvidia-smi SM clock / throttle sampling in the background."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------- roofline bytes ---

def gather_bytes(pattern: np.ndarray, esz: int) -> tuple[int, int]:
    """(sector bytes, element bytes) of one signal's gather at a 32B-aligned base."""
    sectors = np.unique((pattern * esz) // 32).size
    return 32 * sectors, pattern.size * esz


def line_bytes(pattern: np.ndarray, esz: int) -> int:
    """HBM bytes at the measured access granularity: every touched 128 B line
    (profiles/r01_gather_granularity.md)."""
    return 128 * np.unique((pattern * esz) // 128).size


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ------------------------------------------------------------ b200 arm ---

def config_dict(cfg: int, B_total: int, B_rank: int, world: int, scaling: str) -> dict:
    """The workload of a line; byte-identical in both arms (b200 and reference)."""
    from paper_2211_15299_b200 import workloads as W
    spec = W.CONFIGS[cfg]
    k = spec.get("k", 1 << spec["p"])
    return {"workload": f"config {cfg}: N=2^{spec['M']}, k={k}, "
                        + (f"B={B_total} total" if scaling == "strong" else f"B={B_rank} per GPU")
                        + f", {spec['dtype']}, " + ("per-signal supports" if cfg == 4 else "shared support"),
            "global_batch": B_total, "N": 1 << spec["M"], "k": k, "parallelism": f"batch shard x{world}"}


def plan_times_all(S, W, torch, dev, configs) -> dict:
    """Plan build of a fresh SupportSet per config, synchronised: the first
    build (it includes loading the plan kernels of that size) and the median
    of three repeats, before any signal memory is allocated.  The reference rebuilds its plan on every call (hidft.py:154);
    per-signal supports (config 4) derive theirs on chip inside each call, so
    their figure is a one-row call."""
    from paper_2211_15299_b200.hidft import get_plan
    out = {}
    # CUDA context and library initialisation (loading the 15 MB of kernels'
    # module, the first launch) is paid once per process, by whatever call comes
    # first: timed here on an 8-element support and reported as
    # `library_init_ms`, so that `plan_ms` below is the cost of the plan alone
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tiny = S.SupportSet(16, np.array([1, 3, 5, 7, 9, 11, 13, 15], dtype=np.int64))
    get_plan(tiny, S.pivots(tiny), 0, 0, dev)
    torch.cuda.synchronize()
    out["init_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    for cfg in configs:
        spec = W.CONFIGS[cfg]
        cdt = torch.complex64 if spec["dtype"] == "complex64" else torch.complex128
        t = []
        for _ in range(4):  # the first build, then three repeats (their median is the warm figure)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if cfg == 4:
                sup = torch.from_numpy(W.config_supports_batch(4, 1)).to(dev)
                row = torch.zeros((1, 1 << spec["M"]), dtype=cdt, device=dev)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                S.hidft_to_dft_batched(row, sup, check=False)
            else:
                sup, M = W.config_support(cfg)
                J = S.SupportSet(1 << M, sup)  # host validation of the indices is not timed
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                get_plan(J, S.pivots(J), 0, 0 if cdt == torch.complex64 else 1, dev)
            torch.cuda.synchronize()
            t.append((time.perf_counter() - t0) * 1e3)
        out[cfg] = {"cold_ms": round(t[0], 3), "warm_ms": round(sorted(t[1:])[1], 3)}
    torch.cuda.empty_cache()
    return out


def measure_config(args, cfg: int, S, W, torch, dev, rank: int, world: int, dist, steps: int, headline: bool,
                   plan_times: dict):
    """Device-timed steps of one config on this rank; returns (result dict,
    state for the e2e / peer legs).  The caller holds the barrier discipline."""
    spec = W.CONFIGS[cfg]
    if args.scaling == "strong":  # fixed total batch, sharded over the ranks
        from paper_2211_15299_b200.dist import shard_range
        B_total = (args.batch if headline and args.batch else spec["B"])
        b0, b1 = shard_range(B_total, rank, world)
        B = b1 - b0
        if B < 1:
            raise SystemExit(f"strong scaling: {B_total} signals cannot feed {world} ranks")
    else:  # fixed batch per rank
        B = args.batch if headline and args.batch else spec["B"]
        b0, B_total = rank * B, B * world
    wl = W.make_workload(cfg, B, b0=b0)
    cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
    esz = 8 if cdt == torch.complex64 else 16
    N = wl.N

    # byte accounting of one step: 32 B sectors and 128 B lines of the gather
    L2 = 126 * 2 ** 20
    per_sig_sector, lines, ub_sum = [], 0, 0
    if wl.support.ndim == 1:
        piv = S.pivots(S.SupportSet(N, wl.support))
        pat = S.pivoted_pattern(piv, wl.M).as_array()
        gb, ub = gather_bytes(pat, esz)
        per_sig_sector = [gb] * B
        ub_sum = ub * B
        lines = B * line_bytes(pat, esz)
    else:
        for b in range(B):
            pat = W.pattern_of(W.config_pivots(cfg, b0 + b), wl.M)
            gb, ub = gather_bytes(pat, esz)
            per_sig_sector.append(gb)
            ub_sum += ub
            lines += line_bytes(pat, esz)
    if wl.support.ndim == 1:
        J = S.SupportSet(N, wl.support)
    else:
        J = torch.from_numpy(wl.support).to(dev)
    plan_ms = plan_times.get(cfg, {}).get("cold_ms")

    footprint = sum(per_sig_sector)
    R = max(2, math.ceil(4 * L2 / max(footprint, 1)))
    R = min(R, args.max_sets)
    sig_bytes = B * N * esz
    free = torch.cuda.mem_get_info(dev)[0]
    R = max(1, min(R, int((free * 0.85 - 2 * (1 << 30)) // sig_bytes)))
    sets = [torch.empty((B, N), dtype=cdt, device=dev) for _ in range(R)]
    W.synthesize_into(sets[0], wl.support, wl.coeffs)
    for st_ in sets[1:]:
        st_.copy_(sets[0])
    out = torch.empty((B, wl.k), dtype=cdt, device=dev)
    status = torch.zeros(wl.support.shape[0] if wl.support.ndim == 2 else 1, dtype=torch.int32, device=dev)

    # kernels one step launches (the split transforms launch 2-3 per row chunk)
    launches_per_step = 1
    if wl.support.ndim == 1:
        import ctypes
        from paper_2211_15299_b200 import _lib
        from paper_2211_15299_b200.hidft import get_plan
        lp = get_plan(J, S.pivots(J), 0, _lib.C64 if cdt == torch.complex64 else _lib.C128, dev)
        n_l = ctypes.c_int64(0)
        _lib.check(_lib.load().sfft_launch_count(lp.handle, B, ctypes.byref(n_l)))
        launches_per_step = int(n_l.value)

    if cfg == 3:  # sas_transform(f, J, r=pivots(J)): the mu*=1 read, x N/|I|
        r_sas = S.pivots(J)

        def step(i):
            res = S.sas_transform(sets[i % R], J, r=r_sas)
            out.copy_(res.coeffs)
    else:
        def step(i):
            S.hidft_to_dft_batched(sets[i % R], J, out=out, status=status, check=False)

    # correctness gate on the measured configuration: planted spectrum recovered
    step(0)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    err = float(np.max(np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)))
    tol = 1e-5 if esz == 8 else 1e-11
    worst = int(status.max().item())
    if not (err < tol) or worst != 0:
        raise SystemExit(f"bench parity gate failed on config {cfg}: rel L2 {err:.3e} status {worst}")

    # CUDA graphs captured from the same step calls inside a PDL chain scope
    # (S.stream_chain: consecutive library calls on the capture stream may
    # overlap through programmatic dependent launch, as back-to-back eager
    # calls in a scope do): one graph of GS >= --graph-steps consecutive
    # steps (whole cycles over the R rotation sets), one graph for each tail
    # length this run needs, and one graph per single step as a fallback.
    # --no-graph times eager calls (in a scope as well).
    GS = 0

    def run_steps(n, start=0):
        with S.stream_chain():
            for i in range(start, start + n):
                step(i)
    if not args.no_graph:
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for i in range(R):
                step(i)
        torch.cuda.current_stream(dev).wait_stream(side)

        def capture(idx):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                with S.stream_chain():
                    for i in idx:
                        step(i)
            return g
        graphs = [capture([i]) for i in range(R)]
        GS = R * max(1, math.ceil(args.graph_steps / R))  # steps per group graph, whole rotation cycles
        group = capture(range(GS))
        tails = {n: capture(range(n)) for n in {steps % GS, args.warmup % GS, 64 % GS} - {0}}
        torch.cuda.synchronize()

        def run_steps(n, start=0):
            i = start
            while i < start + n:
                left = start + n - i
                if i % GS == 0 and left >= GS:
                    group.replay()
                    i += GS
                elif i % GS == 0 and left in tails:
                    tails[left].replay()
                    i += left
                else:
                    graphs[i % R].replay()
                    i += 1

    local = env_int("LOCAL_RANK", 0)
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    sampler = ClockSampler(vis[local] if local < len(vis) else local)
    sampler.start()
    # soak so that clock samples exist under load, then W warm-up steps
    t_end = time.time() + (args.soak if headline else min(args.soak, 0.5))
    i = 0
    while time.time() < t_end:
        run_steps(64, i)
        i += 64
        torch.cuda.synchronize()
    run_steps(args.warmup)
    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    run_steps(steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    clocks = sampler.stop()
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")
    ms_t = torch.tensor([ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / steps
    coeffs_per_step = B_total * wl.k
    value = coeffs_per_step / (ms_per_step / 1e3)

    # roofline of the step (HBM-bound): G = gather sectors +
    # coefficient writes + support reads (shared: once; per-signal: B*k int64)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    G = footprint + B * wl.k * esz + wl.support.size * 8
    achieved = G / (ms_per_step / 1e3) / 1e9
    A_sl = 1 << (len(S.pivots(J)) if wl.support.ndim == 1 else int(math.log2(wl.k)))
    flops_step = int(B * 5 * A_sl * max(1, int(math.log2(A_sl))))
    fp = fma_peaks()
    fpk = fp["fp32_tflops"] if esz == 8 else fp["fp64_tflops"]
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": None, "peak_source": peak_src,
            "kernels_per_step": launches_per_step,
            "flops": {"per_step": flops_step, "achieved_tflops": round(flops_step / (ms_per_step / 1e3) / 1e12, 3),
                      "peak_tflops": fpk, "peak_source": fp["source"],
                      "frac": round(flops_step / (ms_per_step / 1e3) / 1e12 / fpk, 4)},
            "algorithmic_bytes_per_launch": int(G),
            "element_bytes_per_launch": int(ub_sum + B * wl.k * esz),
            "sector_efficiency": round(ub_sum / max(footprint, 1), 4)}
    # the same step against HBM bytes at the measured 128 B access granularity
    G_line = lines + B * wl.k * esz + wl.support.size * 8
    roof["at_measured_granularity"] = {
        "bytes_per_launch": int(G_line), "achieved": round(G_line / (ms_per_step / 1e3) / 1e9, 1),
        "frac": round(G_line / (ms_per_step / 1e3) / 1e9 / hbm, 4),
        "note": "every isolated HBM read moves a 128 B line on this B200 (profiles/r01_gather_granularity.md)"}
    n_samples = ub_sum / esz
    if lines / 128 >= 0.99 * n_samples:  # every sample in its own line (configs 2-4)
        floor_us = (lines / 128) / 3.94e10 * 1e6
        roof["isolated_line_floor"] = {"us_per_launch": round(floor_us, 2),
                                       "frac": round(floor_us / (ms_per_step * 1e3), 4)}
    tr = profile_traffic(cfg)
    if tr:
        roof["traffic"] = tr.get("traffic")
        roof["traffic_source"] = tr.get("source")
        if tr.get("sector_efficiency_ncu") is not None:
            roof["sector_efficiency_ncu"] = tr["sector_efficiency_ncu"]
    res = {"config": config_dict(cfg, B_total, B, world, args.scaling), "value": value, "ms_per_step": ms_per_step,
           "steps": steps, "gpu_launches": steps * launches_per_step, "roofline": roof, "clocks": clocks,
           "plan_ms": plan_ms, "plan_warm_ms": plan_times.get(cfg, {}).get("warm_ms"),
           "parity": {"rel_l2_vs_planted_max": err, "tol": tol, "status_max": worst, "rows": B},
           "method": {"launch": "eager calls in a stream_chain scope" if args.no_graph else (
                          f"CUDA graphs of {GS} consecutive step calls (rotating over the input sets), "
                          "programmatic dependent launch between steps inside S.stream_chain"),
                      "l2": f"rotating {R} input sets, gather footprint {R * footprint / 2**20:.0f} MiB "
                            f"vs 126 MB L2"}}
    state = {"sets": sets, "J": J, "wl": wl, "esz": esz, "B": B, "B_total": B_total, "status": status,
             "cdt": cdt, "out": out, "coeffs_per_step": coeffs_per_step, "cdev": cdev}
    return res, state


def measure_interleaved(args, cfg: int, S, W, torch, dev, steps: int) -> dict:
    """The same transform on the batch stored sample-major ((N, B): column b =
    signal b, sfft_hidft_interleaved): each needed sample index of a CTA's
    signals is one contiguous run, so G (32 B sectors) equals the element
    bytes.  Secondary line beside the (B, N) headline."""
    spec = W.CONFIGS[cfg]
    B = args.batch or spec["B"]
    wl = W.make_workload(cfg, B)
    cdt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
    esz = 8 if cdt == torch.complex64 else 16
    J = S.SupportSet(wl.N, wl.support)
    piv = S.pivots(J)
    A = 1 << len(piv)
    step_bytes = A * B * esz
    # L2: one copy of the batch, the steps rotate over R shifts; the pattern's
    # offsets are multiples of q = 2^(M-1-r_max), so shifts 0..q-1 read
    # disjoint sample rows (config 2: q = 32, 32 x 8 MiB of rows vs 126 MB L2)
    q = 1 << (wl.M - 1 - piv[-1])
    R = max(1, min(q, 64))
    rows = torch.empty((B, wl.N), dtype=cdt, device=dev)
    W.synthesize_into(rows, wl.support, wl.coeffs)
    nb = rows.T.contiguous()
    del rows
    out = torch.empty((B, wl.k), dtype=cdt, device=dev)
    S.hidft_to_dft_interleaved(nb, J, out=out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    err = float(np.max(np.linalg.norm(got - wl.coeffs, axis=1) / np.linalg.norm(wl.coeffs, axis=1)))
    tol = 1e-5 if esz == 8 else 1e-11
    if not err < tol:
        raise SystemExit(f"interleaved parity gate failed: rel L2 {err:.3e}")
    GS = R * max(1, math.ceil(args.graph_steps / R))
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for i in range(R):
            S.hidft_to_dft_interleaved(nb, J, out=out, shift=i)
    torch.cuda.current_stream(dev).wait_stream(side)
    with torch.cuda.graph(g):
        with S.stream_chain():
            for i in range(GS):
                S.hidft_to_dft_interleaved(nb, J, out=out, shift=i % R)
    reps = max(1, steps // GS)
    for _ in range(max(1, args.warmup // GS + 1)):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (reps * GS)
    hbm = float(measured_peaks().get("hbm_gbs", 6650.0))
    G = step_bytes + B * wl.k * esz + wl.support.size * 8
    ach = G / (ms / 1e3) / 1e9
    del nb
    torch.cuda.empty_cache()
    return {"layout": "(N, B) sample-major: sample n of signal b at n * B + b (sfft_hidft_interleaved)",
            "value": B * wl.k / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "steps": reps * GS,
            "gpu_launches": reps * GS,
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "algorithmic_bytes_per_launch": int(G),
                         "note": "gather runs of 8 signals (64 B): G at 32 B sectors = element bytes"},
            "parity": {"rel_l2_vs_planted_max": err, "tol": tol},
            "l2": f"rotating {R} shifts reading disjoint sample rows, {R * step_bytes / 2**20:.0f} MiB of gathered "
                  f"samples per cycle vs 126 MB L2"}


_FMA_LIVE: dict | None = None


def fma_peaks() -> dict:
    """Non-tensor FMA peaks measured in this run (sfft_probe_fma_peak: FMA
    chains on every SM, CUDA events, once per process, outside every timed
    region); profiles/fma_peak.json (tools/fma_peak.cu on the GPU box,
    committed) when the probe is unavailable."""
    global _FMA_LIVE
    if _FMA_LIVE is None:
        try:
            import ctypes
            from paper_2211_15299_b200 import _lib
            lib = _lib.load()
            out = {}
            for name, code in (("fp32_tflops", 0), ("fp64_tflops", 1)):
                v = ctypes.c_double(0.0)
                _lib.check(lib.sfft_probe_fma_peak(code, ctypes.byref(v), _lib.stream_ptr()))
                out[name] = round(float(v.value), 2)
            out["source"] = "measured in this run (sfft_probe_fma_peak: FMA chains on every SM, CUDA events)"
            _FMA_LIVE = out
        except Exception:  # noqa: BLE001  (no device / older library: the committed measurement)
            _FMA_LIVE = {}
    if _FMA_LIVE:
        return _FMA_LIVE
    try:
        with open(os.path.join(ROOT, "profiles", "fma_peak.json")) as fh:
            d = json.load(fh)
        return {"fp32_tflops": float(d["fp32_tflops"]), "fp64_tflops": float(d["fp64_tflops"]),
                "source": "profiles/fma_peak.json (tools/fma_peak.cu, measured on the B200 box)"}
    except (OSError, ValueError, KeyError):
        return {"fp32_tflops": 66.4, "fp64_tflops": 32.7, "source": "round-1 tools/fma_peak.cu measurement"}


def profile_traffic(cfg: int) -> dict | None:
    """ncu-measured DRAM traffic per step and sector efficiency (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            d = json.load(fh)
    except (OSError, ValueError):
        return None
    e = d.get(f"cfg{cfg}")
    if e is None:
        return None
    if not isinstance(e, dict):
        return {"traffic": e, "source": "profiles/traffic.json (ncu dram__bytes_read+write)"}
    return {"traffic": e.get("traffic"), "source": e.get("source", "profiles/traffic.json"),
            "sector_efficiency_ncu": e.get("sector_efficiency_ncu")}


def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_2211_15299_b200 as S
    from paper_2211_15299_b200 import workloads as W

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    ndev = torch.cuda.device_count()
    local_world = env_int("LOCAL_WORLD_SIZE", world)
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device")
    if args.dist_backend == "nccl" and local_world > ndev:
        raise SystemExit(f"bench.py: --gpus {world} needs {local_world} devices on this node, found {ndev}")
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:  # host-side collectives only (CPU tests of the multi-rank path)
            dist.init_process_group("gloo")

    configs = [args.config] + ([c for c in (1, 2, 3, 4, 5, 6) if c != args.config]
                               if world == 1 and not args.no_per_config else [])
    plan_times = plan_times_all(S, W, torch, dev, configs)
    head, st = measure_config(args, args.config, S, W, torch, dev, rank, world, dist, args.steps, True, plan_times)

    # N > 1, timed: one step with the result rows written straight into
    # rank 0's device buffer over peer memory (dist.PeerRows),
    # checked on rank 0 against the planted spectra of every rank's first and
    # last row; the timed steps above leave the rows sharded
    peer_info = None
    if world > 1 and args.config != 3 and not args.no_peer_gather:
        peer_info = run_peer_gather(S, W, torch, dist, st["sets"][0], st["J"], st["wl"], args.config, st["B"],
                                    st["B_total"], st["status"], st["cdt"], rank, world)

    # end to end through the public API with host buffers (rank-local)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, S, torch, st["sets"][0], st["J"], st["wl"], st["esz"], dev)
        if world > 1:
            t = torch.tensor([e2e["seconds_per_step"]], dtype=torch.float64, device=st["cdev"])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["value"] = st["coeffs_per_step"] / float(t.item())
        del e2e["seconds_per_step"]
    del st
    torch.cuda.empty_cache()

    layouts = {}
    if world == 1 and not args.no_per_config and args.config in (1, 2):
        try:
            layouts["interleaved"] = measure_interleaved(args, args.config, S, W, torch, dev, args.steps)
        except SystemExit as e:
            layouts["interleaved"] = {"error": str(e)}

    # every other config on the record (N = 1): same discipline, same run
    per_config = {}
    if world == 1 and not args.no_per_config:
        for c in [c for c in (1, 2, 3, 4, 5, 6) if c != args.config]:
            steps_c = max(20, min(args.steps, args.per_config_steps))
            try:
                r, stc = measure_config(args, c, S, W, torch, dev, rank, world, dist, steps_c, False, plan_times)
                del stc
                if not args.no_cpu:
                    r["reference_single_call"] = reference_single_call(c)
                per_config[f"cfg{c}"] = r
            except SystemExit as e:  # a failed parity gate is reported, not hidden
                per_config[f"cfg{c}"] = {"error": str(e)}
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = run_cpu_reference(args.config, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None,
            "dtype": "c64 (f32)" if W.CONFIGS[args.config]["dtype"] == "complex64" else "c128 (f64)",
            "data": "synthetic: seeded supports (reference generators) and complex-Gaussian spectra, "
                    "signals = inverse DFT synthesised on device",
            "config": head["config"],
            "method": head["method"],
            "gpu_launches": head["gpu_launches"],
            "roofline": head["roofline"],
            "clocks": head["clocks"],
            "plan_ms": head["plan_ms"], "plan_warm_ms": head["plan_warm_ms"],
            "library_init_ms": plan_times.get("init_ms"),
            "parity": head["parity"],
        }
        if e2e:
            line["e2e"] = e2e
        if peer_info:
            line["peer_gather"] = peer_info
        if cpu:
            line["cpu_baseline"] = cpu
        if layouts:
            line["layouts"] = layouts
        if per_config:
            line["per_config"] = per_config
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_peer_gather(S, W, torch, dist, signals, J, wl, cfg, B, B_total, status, cdt, rank, world) -> dict:
    """One step per rank writing its rows into rank 0's buffer through CUDA
    IPC peer memory (the transform's own epilogue stores); device time max
    over ranks; rank 0 checks rows against the planted spectra.  Failures are
    reported in the line, not raised (the timed numbers stand on their own)."""
    from paper_2211_15299_b200.dist import PeerRows, shard_range
    try:
        peer = PeerRows(B_total, wl.k, cdt)  # collective; raises on every rank together
        fits = torch.tensor([1 if peer.rows[1] - peer.rows[0] == B else 0], dtype=torch.int32)
        if dist.get_backend() == "nccl":
            fits = fits.cuda()
        dist.all_reduce(fits, op=dist.ReduceOp.MIN)
        if int(fits.item()) == 0:
            peer.close()
            return {"error": "peer rows do not match the ranks' signal shards"}
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.hidft_to_dft_batched(signals, J, out=peer.local, status=status, check=False)
        e1.record()
        full = peer.complete()
        ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64)
        if dist.get_backend() == "nccl":
            ms = ms.cuda()
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        info = {"rows": B_total, "ms_step": round(float(ms.item()), 4), "status_max": int(status.max().item()),
                "path": "dist.PeerRows: rank 0 exports a CUDA IPC handle of its B x k result buffer; every "
                        "rank's transform stores its row shard there over NVLink/NVSwitch peer memory"}
        if rank == 0:
            errs = []
            for r in range(world):
                a, b = shard_range(B_total, r, world)
                for row in sorted({a, b - 1}):
                    want = W.make_workload(cfg, B=1, b0=row).coeffs[0]
                    got = full[row].cpu().numpy()
                    errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
            info["rows_checked"] = len(errs)
            info["max_rel_l2"] = max(errs)
        peer.close()
        return info
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)[:300]}


def run_e2e(args, S, torch, dev_signals, J, wl, esz, dev) -> dict:
    """Public API, host buffers: signals in page-locked host memory (zero-copy
    gather of the 2^s needed samples per signal over PCIe), per-signal
    supports (config 4) copied from pinned host memory every step, and the
    coefficients returned to host memory; every step synchronises."""
    host = torch.empty(dev_signals.shape, dtype=dev_signals.dtype, pin_memory=True)
    host.copy_(dev_signals)
    torch.cuda.synchronize()
    B = dev_signals.shape[0]
    support_bytes = 0
    if wl.cfg == 3:
        r_sas = S.pivots(J)
        A = 1 << len(r_sas)

        def call():
            return S.sas_transform(host, J, r=r_sas).coeffs
    elif wl.support.ndim == 2:
        hostJ = torch.from_numpy(wl.support).pin_memory()
        support_bytes = hostJ.numel() * 8
        A = wl.support.shape[1]

        def call():
            return S.hidft_to_dft_batched(host, hostJ)
    else:
        A = wl.k

        def call():
            return S.hidft_to_dft_batched(host, J)
    res = None
    for _ in range(max(3, args.warmup)):  # same pattern as the timed loop: warms the pinned host cache
        res = call()
    steps = max(3, min(args.steps, args.e2e_steps))
    per = []
    t0 = time.perf_counter()
    for _ in range(steps):
        t1 = time.perf_counter()
        res = call()
        per.append(time.perf_counter() - t1)
    dt = (time.perf_counter() - t0) / steps
    print(f"e2e per-step ms: min {min(per) * 1e3:.3f} median {sorted(per)[len(per) // 2] * 1e3:.3f} "
          f"max {max(per) * 1e3:.3f}", file=sys.stderr)
    del host
    return {"value": B * wl.k / dt, "unit": UNIT, "h2d_bytes_per_step": int(B * A * esz + support_bytes),
            "d2h_bytes_per_step": int(np.asarray(res).size * esz), "seconds_per_step": dt,
            "path": ("public API on page-locked host rows and supports -> sfft_hidft_to_dft_fused_host: host "
                     "threads derive each support's pivots and gather its 2^s samples while earlier row chunks "
                     "(samples + supports) are copied, transformed with on-chip plans and copied back"
                     if wl.support.ndim == 2 else
                     "public API on a page-locked host tensor -> sfft_hidft_host: native host threads gather "
                     "the 2^s needed samples per signal into pinned staging while earlier row chunks are "
                     "copied to the device, transformed and copied back (downloads on a second stream)")}


# ------------------------------------------------------- CPU reference ---

def _reference_module():
    """The unmodified reference package from baseline/_ref (pip install
    --target baseline/_ref /root/reference/pkg), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "structfft")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import structfft  # noqa: F401
        return structfft
    except Exception:  # noqa: BLE001
        return None


def _reference_callables(cfg: int):
    """(kind, prepare(J, M) -> support object, call(f, Jobj)) of the CPU leg:
    the reference's public path (hidft.py:135-207, sas.py:313-409) when
    installed, else the oracle port of it."""
    sf = _reference_module()
    if sf is not None:
        def prep(J, M):
            return sf.SupportSet.make(1 << M, J.tolist())
        if cfg == 3:
            def call(f, Js):
                return sf.sas_transform(f, Js, r=sf.pivots(Js)).coeffs
        else:
            def call(f, Js):
                return sf.hidft_to_dft(sf.hidft(f, Js, sf.pivots(Js)))
        return "reference", prep, call
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import structfft_oracle as O

    def prep(J, M):
        return (J, M)
    if cfg == 3:
        def call(f, Js):
            return O.reference_sas_call(f, Js[0], Js[1])
    else:
        def call(f, Js):
            return O.reference_call(f, Js[0], Js[1])
    return "port", prep, call


def _host_signal(cfg: int, b: int):
    """Signal b of config cfg as a dense host array of the config dtype
    (harness: the oracle's synthesis, the inverse DFT of the spectrum)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import structfft_oracle as O
    from paper_2211_15299_b200 import workloads as W
    spec = W.CONFIGS[cfg]
    J, M = W.config_support(cfg, b)
    coef = W.coefficients(cfg, b, J.size)
    f = O.synthesize(J, coef, M).astype(np.complex64 if spec["dtype"] == "complex64" else np.complex128)
    return J, M, f, coef


def reference_single_call(cfg: int) -> dict:
    """One core, one signal: the reference call's wall time (after one
    warm-up call) and, when the reference is installed, the port's time on
    the same signal (their ratio shows how faithful the port is in cost)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    kind, prep, call = _reference_callables(cfg)
    J, M, f, coef = _host_signal(cfg, 0)
    Js = prep(J, M)
    call(f, Js)
    t0 = time.perf_counter()
    got = call(f, Js)
    dt = time.perf_counter() - t0
    err = float(np.linalg.norm(np.asarray(got) - coef) / np.linalg.norm(coef))
    info = {"kind": kind, "ms_per_signal": round(dt * 1e3, 3), "coeffs_per_s_per_core": J.size / dt,
            "rel_l2_vs_planted": err}
    if kind == "reference":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import structfft_oracle as O
        port = O.reference_sas_call if cfg == 3 else O.reference_call
        port(f, J, M)
        t0 = time.perf_counter()
        port(f, J, M)
        info["port_ms_per_signal"] = round((time.perf_counter() - t0) * 1e3, 3)
        info["port_over_reference_time"] = round(info["port_ms_per_signal"] / info["ms_per_signal"], 3)
    return info


def _cpu_worker(cfg, rows, steps, barrier, queue):
    """One host process: synthesise its rows (untimed), then time `steps`
    passes of the reference call over them, each pass starting on a barrier."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    kind, prep, call = _reference_callables(cfg)
    sigs = []
    for b in rows:
        J, M, f, _ = _host_signal(cfg, b)
        sigs.append((prep(J, M), f, J.size))
    ncoef = sum(k for _, _, k in sigs)
    for step in range(steps):
        barrier.wait()
        t0 = time.perf_counter()
        for Js, f, _ in sigs:
            call(f, Js)
        queue.put((step, time.perf_counter() - t0, ncoef))


def cpu_reference_steps(cfg: int, steps: int, seconds: float) -> tuple[list, dict]:
    """The reference call on every host core, one process per core (the
    reference's own process-pool mechanism, bench.py:261-263).  Each step is
    a bounded sample: every worker runs its rows once; step value =
    coefficients / slowest worker's time."""
    import multiprocessing as mp
    from paper_2211_15299_b200 import workloads as W
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    P = os.cpu_count() or 1
    spec = W.CONFIGS[cfg]
    kind, prep, call = _reference_callables(cfg)
    J, M, f0, _ = _host_signal(cfg, 0)
    esz = f0.itemsize
    Js = prep(J, M)
    call(f0, Js)
    t0 = time.perf_counter()
    call(f0, Js)
    per_sig = time.perf_counter() - t0
    del f0
    mem_rows = max(1, (1 << 30) // ((1 << M) * esz))          # <= 1 GiB of signals per worker
    time_rows = max(1, int(seconds / max(steps, 1) / per_sig))  # bounded step time
    per_worker = max(1, min(mem_rows, time_rows, -(-spec["B"] // P)))
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(P)
    queue = ctx.Queue()
    procs = []
    for w in range(P):
        rows = [(w * per_worker + i) % spec["B"] for i in range(per_worker)]
        procs.append(ctx.Process(target=_cpu_worker, args=(cfg, rows, steps, barrier, queue)))
    t_wall = time.perf_counter()
    for p in procs:
        p.start()
    per_step = {}
    for _ in range(P * steps):
        step, dt, n = queue.get(timeout=3600)
        slot = per_step.setdefault(step, [0.0, 0])
        slot[0] = max(slot[0], dt)
        slot[1] += n
    for p in procs:
        p.join(timeout=60)
    vals = [per_step[s][1] / per_step[s][0] for s in range(steps)]
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    what = ("unmodified reference structfft (baseline/_ref)" if kind == "reference"
            else "oracle port of the reference call (baseline/_ref absent)")
    info = {"unit": UNIT, "cores": P, "kind": kind,
            "sample": f"{P * per_worker} signals of config {cfg} per step ({per_worker} per worker process, "
                      f"{P} processes on {model or 'host CPU'}); {what}: "
                      f"{'sas_transform(f, J, r=pivots(J))' if cfg == 3 else 'hidft(f, J, pivots(J)) + hidft_to_dft'}"
                      f" on dense host arrays of the config dtype; single-call probe {per_sig * 1e3:.2f} ms/signal; "
                      f"total wall {time.perf_counter() - t_wall:.1f} s"}
    return vals, info


def run_cpu_reference(cfg: int, seconds: float) -> dict:
    vals, info = cpu_reference_steps(cfg, 2, seconds)
    return {"value": vals[-1], **info}


def run_reference(args) -> None:
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    world = env_int("WORLD_SIZE", 1)
    cfg = args.config
    from paper_2211_15299_b200 import workloads as W
    vals, info = cpu_reference_steps(cfg, args.warmup + args.steps, args.ref_seconds)
    timed = vals[args.warmup:]
    value = statistics.median(timed)
    spec = W.CONFIGS[cfg]
    k = spec.get("k", 1 << spec["p"])
    B = args.batch or spec["B"]
    B_total = B if args.scaling == "strong" else B * world
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": B_total * k / value * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "c64 input, f64 compute (reference upcasts)" if spec["dtype"] == "complex64" else "c128 (f64)",
            "data": "synthetic, same seeds as the b200 arm",
            "config": config_dict(cfg, B_total, B, world, args.scaling),
            "cpu_baseline": {"value": value, **info},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if info["kind"] == "reference":
        try:
            line["port_check"] = reference_single_call(cfg)
        except Exception as e:  # noqa: BLE001
            line["port_check"] = {"error": repr(e)[:200]}
    print(json.dumps(line), flush=True)


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: re-run this script with N ranks under
    torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="GPUs (ranks); > 1 outside torchrun re-launches under it")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5, 6])
    ap.add_argument("--batch", type=int, default=0,
                    help="signals per GPU (weak) or in total (strong); default: the config's B")
    ap.add_argument("--no-graph", action="store_true", help="time eager calls instead of CUDA-graph replays")
    ap.add_argument("--graph-steps", type=int, default=32, help="steps captured per group graph (rounded up to "
                    "whole rotation cycles)")
    ap.add_argument("--scaling", choices=("weak", "strong"), default="weak",
                    help="weak: the config's B per GPU (default); strong: the config's B split over the GPUs")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--max-sets", type=int, default=8)
    ap.add_argument("--soak", type=float, default=1.0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--per-config-steps", type=int, default=100, help="timed steps of each per_config entry")
    ap.add_argument("--no-per-config", action="store_true", help="headline config only")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="CPU-baseline budget (b200 arm)")
    ap.add_argument("--ref-seconds", type=float, default=150.0, help="whole --impl reference run budget")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-peer-gather", action="store_true", help="N > 1: skip the peer-memory gather step")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-side collectives (multi-rank path test on fewer GPUs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = env_int("WORLD_SIZE", 0)
    if args.gpus is not None and args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if world == 0 and args.gpus and args.gpus > 1:
        raise SystemExit(relaunch(args))
    if world and args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
