"""The Hi-DFT on B200: reference hidft.py's API over the CUDA C-ABI.

`hidft(source, J, r, height, shift)` and `hidft_to_dft(res)` keep the
reference signatures and results (hidft.py:135-207); a source may now also be
a (B, N) batch.  `hidft_to_dft_batched` is the batched hot path: for a shared
support one launch gathers the 2^s samples of every signal through the
support's cached device plan, runs the butterfly and writes (Ff)_J in
ascending-J order; for per-signal supports one fused launch also derives each
signal's plan on chip.

Sources (hidft.py:34-49):
  * CUDA tensor (N,) or (B, N), complex64 / complex128 -> computed in that
    precision (complex64 signals run the float32 kernels);
  * host-resident numpy / CPU tensor (pinned or pageable) -> the library's
    host thread pool gathers the 2^s samples per signal into pinned staging
    (deriving per-signal pivots on the host for per-signal supports),
    pipelined with their DMA, the device transform and the copy back: only
    those samples cross PCIe;
  * callable loc -> samples, or an object with `sample_block(loc)` (e.g. the
    reference's BandlimitedSignal) -> evaluated at the plan's offsets on the
    host (band-limited sources are synthesised on the device), then
    transformed on the device.
Results are CUDA tensors for CUDA sources and host arrays otherwise.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np

from . import _lib
from .congruence import (SupportSet, as_support, classify, validate_pivot_vector)
from .errors import ContractViolationError, InvalidInputError

_DT = {}  # filled lazily: torch dtype -> C dtype code


def _torch():
    import torch
    if not _DT:
        _DT[torch.complex64] = _lib.C64
        _DT[torch.complex128] = _lib.C128
    return torch


# ------------------------------------------------------------------ plans ---

class ButterflyPlan:
    """Device ButterflyPlan (hidft.py:52-95) for one (J, used pivots, dtype).

    Built by sfft_plan_create; the tables stay in HBM.  Host copies of the
    index tables are made on demand (bit-exact with the reference)."""

    def __init__(self, J: SupportSet, r: tuple[int, ...], height: int, dtype_code: int, device):
        lib = _lib.load()
        self.support = J
        self.device = device
        self.dtype_code = dtype_code
        self._lib = lib
        self.handle = ctypes.c_void_p(0)
        rr = np.asarray(r if r else [0], dtype=np.int32)
        dj = J.device_tensor(device)
        with _torch().cuda.device(device):  # the plan belongs to the current device
            _lib.check(lib.sfft_plan_create(dj.data_ptr(), len(J), J.M, rr.ctypes.data, len(r), int(height),
                                            dtype_code, _lib.stream_ptr(device), ctypes.byref(self.handle)))
        info = _lib.PlanInfo()
        _lib.check(lib.sfft_plan_get_info(self.handle, ctypes.byref(info)))
        self.r = tuple(r)
        self.height = int(height)
        self.s = info.s
        self.used = tuple(int(info.used[i]) for i in range(info.s))
        self.level = info.level
        self.A = int(info.A)
        self.k = int(info.k)
        self.n_nodes = int(info.n_nodes)
        self.mu_star = int(info.mu_star)
        self.homogeneous = bool(info.homogeneous)
        self.pivot_mask = int(info.pivot_mask)
        self._tables = None

    @property
    def n_slots(self) -> int:
        return self.A

    def tables(self) -> dict[str, np.ndarray]:
        """element_slots, slot_residues, slot_real, node_residues, offsets,
        twiddles -- copied from the device."""
        if self._tables is None:
            k, A, n = self.k, self.A, self.n_nodes
            es = np.empty(k, np.int64)
            sr = np.empty(A, np.int64)
            real = np.empty(A, np.uint8)
            nr = np.empty(max(n, 1), np.int64)
            off = np.empty(A, np.int64)
            tw = np.empty(max(A - 1, 1), np.complex64 if self.dtype_code == _lib.C64 else np.complex128)
            _lib.check(self._lib.sfft_plan_tables(self.handle, es.ctypes.data, sr.ctypes.data,
                                                  real.ctypes.data, nr.ctypes.data, off.ctypes.data,
                                                  tw.ctypes.data, _lib.stream_ptr(self.device)))
            self._tables = {"element_slots": es, "slot_residues": sr, "slot_real": real.astype(bool),
                            "node_residues": nr[:n], "offsets": off, "twiddles": tw[: A - 1]}
        return self._tables

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.sfft_plan_destroy(h)
            except Exception:
                pass
            h.value = None


def get_plan(J: SupportSet, r: tuple[int, ...], height: int, dtype_code: int, device) -> ButterflyPlan:
    """Plan cache on the immutable support (SPEC.md:342 allows caching)."""
    key = (tuple(r), int(height), dtype_code, str(device))
    plan = J._plans.get(key)
    if plan is None:
        plan = ButterflyPlan(J, tuple(r), height, dtype_code, device)
        J._plans[key] = plan
    return plan


# ---------------------------------------------------------------- sources ---

@dataclass
class _Src:
    kind: str               # "device" | "host" | "callable" | "synth"
    tensor: Any = None      # 2-D (B, N) view for device/host
    batched: bool = False
    dtype_code: int = _lib.C128
    device: Any = None
    fn: Any = None


def _prepare_source(source, N: int) -> _Src:
    torch = _torch()
    dev = _lib.require_device()
    if isinstance(source, torch.Tensor):
        t = source
        if not t.is_complex():
            t = t.to(torch.complex128)
        if t.dtype not in _DT:
            raise InvalidInputError(f"unsupported signal dtype {t.dtype}")
        if t.dim() not in (1, 2) or t.shape[-1] != N:
            raise InvalidInputError("dense signal must be a length-N vector or a (B, N) batch")
        batched = t.dim() == 2
        t2 = t if batched else t.unsqueeze(0)
        if t2.stride(-1) != 1:
            t2 = t2.contiguous()
        if t2.is_cuda:
            return _Src("device", t2, batched, _DT[t2.dtype], t2.device)
        return _Src("host", t2, batched, _DT[t2.dtype], dev)  # gathered on the host, see _host_gather
    if hasattr(source, "support") and hasattr(source, "coeffs") and hasattr(source, "sample_block"):
        # BandlimitedSignal (ours or the reference's): synthesise on the device
        from .signals import BandlimitedSignal
        if int(source.N) != N:
            raise InvalidInputError("signal modulus does not match support")
        return _Src("synth", None, False, _lib.C128, dev, BandlimitedSignal.from_reference(source))
    if callable(source) or hasattr(source, "sample_block"):
        if hasattr(source, "N") and int(getattr(source, "N")) != N:
            raise InvalidInputError("signal modulus does not match support")
        fn = source.sample_block if hasattr(source, "sample_block") else source
        return _Src("callable", None, False, _lib.C128, dev, fn)
    arr = np.asarray(source)
    if arr.dtype != np.complex64:
        arr = np.asarray(arr, dtype=np.complex128)
    if arr.ndim not in (1, 2) or arr.shape[-1] != N:
        raise InvalidInputError("dense signal must be a length-N vector or a (B, N) batch")
    batched = arr.ndim == 2
    t = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1, N)))
    return _Src("host", t, batched, _DT[t.dtype], dev)


def _signal_ptr(src: _Src) -> int:
    return src.tensor.data_ptr()


HOST_GATHER_THREADS = 0   # host gather workers besides the caller; 0: every other core
HOST_CHUNK_ROWS = 0       # rows per pipelined chunk; 0: B/16 (at least 32)


def _host_threads() -> int:
    return HOST_GATHER_THREADS


def _host_transform(sig, plan: "ButterflyPlan", shift: int, out_kind: int, n_out: int, with_slots=False):
    """Transform host-resident rows through sfft_hidft_host: native host
    threads gather each row's 2^s samples into page-locked staging while
    earlier row chunks are copied to the device, transformed
    (sfft_hidft_gathered) and copied back, all on the current stream.
    Returns the (B, n_out) result (and the (B, A) slot values) in pinned host
    memory."""
    torch = _torch()
    lib = _lib.load()
    B = sig.shape[0]
    out_host = torch.empty((B, n_out), dtype=sig.dtype, pin_memory=True)
    slots = torch.empty((B, plan.A), dtype=sig.dtype, pin_memory=True) if with_slots else None
    with torch.cuda.device(plan.device):
        sp = _lib.stream_ptr(plan.device)
        _lib.check(lib.sfft_hidft_host(plan.handle, sig.data_ptr(), B, sig.stride(0), int(shift), out_kind,
                                       out_host.data_ptr(), n_out, slots.data_ptr() if with_slots else None,
                                       plan.A, HOST_CHUNK_ROWS, HOST_GATHER_THREADS, sp))
    return (out_host, slots) if with_slots else out_host


def _gathered_samples(src: _Src, plan: "ButterflyPlan", shift: int):
    """(1, A) complex128 device tensor of the samples at (I - shift) mod N in
    slot order, for sources that are evaluated rather than stored
    (hidft.py:36-45): synthesised on the device for a BandlimitedSignal, or
    the callable's values otherwise."""
    torch = _torch()
    N = plan.support.N
    loc = (plan.tables()["offsets"] - int(shift)) % N
    if src.kind == "synth":
        return src.fn.sample_block_tensor(torch.as_tensor(loc, device=src.device)).view(1, -1)
    vals = np.asarray(src.fn(loc), dtype=np.complex128)
    if vals.shape != loc.shape:
        raise InvalidInputError("sample callback returned wrong shape")
    return torch.from_numpy(vals.reshape(1, -1)).to(src.device)


# ----------------------------------------------------------------- result ---

@dataclass
class HiDftResult:
    """Per-node transform values at one height (hidft.py:98-132).

    node_values / slot_values are (n,) for a single signal or (B, n) for a
    batch; torch CUDA tensors for CUDA sources, numpy otherwise."""

    support: SupportSet
    pivots: tuple[int, ...]
    height: int
    shift: int
    level: int
    node_residues: tuple[int, ...]
    node_values: Any
    slot_values: Any
    slot_residues: np.ndarray
    slot_real: np.ndarray
    ops_adds: int
    ops_mults: int
    plan: ButterflyPlan | None = field(default=None, repr=False)
    on_device: bool = field(default=False, repr=False)

    def _host(self, x) -> np.ndarray:
        return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)

    @property
    def values(self) -> dict:
        vals = self._host(self.node_values)
        if vals.ndim == 1:
            return {int(r): complex(v) for r, v in zip(self.node_residues, vals)}
        return {int(r): vals[:, i] for i, r in enumerate(self.node_residues)}

    def value_at_index(self, j: int):
        res = int(j) % (1 << self.level)
        vals = self.values
        if res not in vals:
            raise InvalidInputError(f"index {j} belongs to no stored node")
        return vals[res]

    def _element_nodes(self) -> np.ndarray:
        res = self.support.as_array() & ((1 << self.level) - 1)
        return np.searchsorted(np.asarray(self.node_residues, np.int64), res)

    def values_by_index(self):
        """One value per support element, in support order (hidft.py:127-132)."""
        idx = self._element_nodes()
        if self.on_device:
            torch = _torch()
            return self.node_values[..., torch.as_tensor(idx, device=self.node_values.device)]
        return np.asarray(self._host(self.node_values))[..., idx].astype(np.complex128)


def _count(counter, A: int, stages: int) -> None:
    if counter is not None and stages:
        for _ in range(stages):  # per stage, as hidft.py:165-167
            counter.mul(A // 2, phase="hidft")
            counter.add(A, phase="hidft")


def _finish(x, src: _Src):
    """Drop the batch axis for single signals; host sources get numpy."""
    if not src.batched:
        x = x[0]
    if src.kind == "device":
        return x
    return x.cpu().numpy()


def _device_guard(x):
    """Make a CUDA tensor argument's device current for the library calls
    (kernels launch on the current device's stream; plans belong to it)."""
    torch = _torch()
    if torch.is_tensor(x) and x.is_cuda:
        return torch.cuda.device(x.device)
    return contextlib.nullcontext()


def hidft(source, J, r: Sequence[int], height: int = 0, shift: int = 0, counter=None) -> HiDftResult:
    """Generalised radix-2 transform of tau^shift f (hidft.py:135-185).

    Output equals F(node representatives, I_{r^{n-}}) applied to the shifted
    samples, unscaled; exactly 1.5*A*log2(A) complex operations are counted."""
    with _device_guard(source):
        return _hidft(source, J, r, height, shift, counter)


def _hidft(source, J, r, height, shift, counter) -> HiDftResult:
    torch = _torch()
    J = as_support(J)
    rt = validate_pivot_vector(r, J.M)
    src = _prepare_source(source, J.N)
    plan = get_plan(J, rt, height, src.dtype_code, src.device)
    cdt = torch.complex64 if src.dtype_code == _lib.C64 else torch.complex128
    lib = _lib.load()
    stream = _lib.stream_ptr(src.device)
    if src.kind in ("callable", "synth"):
        samples = _gathered_samples(src, plan, shift)
        B = 1
        nodes = torch.empty((B, max(plan.n_nodes, 1)), dtype=cdt, device=src.device)
        slots = torch.empty((B, plan.A), dtype=cdt, device=src.device)
        _lib.check(lib.sfft_hidft_gathered(plan.handle, samples.data_ptr(), B, plan.A, _lib.OUT_NODES,
                                           nodes.data_ptr(), nodes.shape[1], slots.data_ptr(), plan.A,
                                           stream))
    elif src.kind == "host":
        sig = src.tensor
        B = sig.shape[0]
        nodes, slots = _host_transform(sig, plan, shift, _lib.OUT_NODES, max(plan.n_nodes, 1), with_slots=True)
    else:
        sig = src.tensor
        B = sig.shape[0]
        nodes = torch.empty((B, max(plan.n_nodes, 1)), dtype=cdt, device=src.device)
        slots = torch.empty((B, plan.A), dtype=cdt, device=src.device)
        _lib.check(lib.sfft_hidft(plan.handle, _signal_ptr(src), B, sig.stride(0), int(shift),
                                  _lib.OUT_NODES, nodes.data_ptr(), nodes.shape[1], slots.data_ptr(),
                                  plan.A, stream))
    nodes = nodes[:, : plan.n_nodes]
    _count(counter, plan.A, plan.s)
    tabs = plan.tables()
    return HiDftResult(
        support=J, pivots=rt, height=int(height), shift=int(shift), level=plan.level,
        node_residues=tuple(int(x) for x in tabs["node_residues"]),
        node_values=_finish(nodes, src), slot_values=_finish(slots, src),
        slot_residues=tabs["slot_residues"].copy(), slot_real=tabs["slot_real"].copy(),
        ops_adds=plan.A * plan.s, ops_mults=(plan.A // 2) * plan.s,
        plan=plan, on_device=src.kind == "device")


def hidft_to_dft(res: HiDftResult, counter=None):
    """(F f)_J from a height-0 transform of a homogeneous support
    (hidft.py:188-207): node values x N/|J| in ascending-J order."""
    torch = _torch()
    J = res.support
    if not classify(J).is_homogeneous:
        raise ContractViolationError("hidft_to_dft requires a homogeneous support")
    if res.height != 0:
        raise ContractViolationError("hidft_to_dft requires a height-0 transform")
    plan = res.plan
    if plan is None:
        raise InvalidInputError("result was not produced by this package's hidft")
    slots = res.slot_values
    host = not torch.is_tensor(slots)
    if host:
        slots = torch.from_numpy(np.ascontiguousarray(slots)).to(plan.device)
    single = slots.dim() == 1
    s2 = slots.unsqueeze(0) if single else slots
    s2 = s2.contiguous()
    out = torch.empty((s2.shape[0], len(J)), dtype=s2.dtype, device=s2.device)
    _lib.check(_lib.load().sfft_plan_apply_map(plan.handle, _lib.OUT_DFT, s2.data_ptr(), s2.shape[0],
                                               s2.shape[1], out.data_ptr(), len(J),
                                               _lib.stream_ptr(plan.device)))
    if counter is not None and J.N != len(J):
        counter.mul(len(J), phase="read")
    if single:
        out = out[0]
    return out.cpu().numpy() if host else out


def _check_out(out, shape, dtype, device, name):
    """A caller-supplied output buffer must match exactly: the C-ABI writes
    through its data pointer and row stride only."""
    torch = _torch()
    if not torch.is_tensor(out):
        raise InvalidInputError(f"{name} must be a tensor")
    if out.dtype != dtype:
        raise InvalidInputError(f"{name} has dtype {out.dtype}, expected {dtype}")
    if out.device != device:
        raise InvalidInputError(f"{name} is on {out.device}, expected {device}")
    if tuple(out.shape) != tuple(shape):
        raise InvalidInputError(f"{name} has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if out.stride(-1) != 1 or (len(shape) == 2 and shape[0] > 1 and out.stride(0) < shape[1]):
        raise InvalidInputError(f"{name} rows must be contiguous and must not overlap")


def hidft_to_dft_batched(signals, J, out=None, status=None, check: bool = True):
    """Fused hidft(f_b, J_b, pivots(J_b)) + hidft_to_dft for a batch.

    signals: (B, N) complex64/complex128 CUDA tensor, or a CPU tensor (the
    needed samples are gathered on the host and the result returned on the
    host; with per-signal supports a page-locked tensor is read zero-copy).
    J: one SupportSet shared by all rows, or a (B, k) int64 tensor with one
    sorted support per row (config 4).  Per-row statuses land in `status`
    (int32 device tensor) when given; with check=True a non-homogeneous or
    invalid support raises like the reference would."""
    with _device_guard(signals):
        return _hidft_to_dft_batched(signals, J, out, status, check)


def _hidft_to_dft_batched(signals, J, out, status, check):
    torch = _torch()
    dev = _lib.require_device()
    if not torch.is_tensor(signals):  # numpy rows stay on the host: only the needed samples move
        signals = torch.from_numpy(np.ascontiguousarray(np.asarray(signals)))
    single = signals.dim() == 1
    sig = signals.unsqueeze(0) if single else signals
    if sig.dtype not in (torch.complex64, torch.complex128):
        raise InvalidInputError("signals must be complex64 or complex128")
    if sig.stride(-1) != 1:
        sig = sig.contiguous()
    B, N = sig.shape
    M = N.bit_length() - 1
    if N & (N - 1):
        raise InvalidInputError(f"N={N} is not a power of two")
    host_out = not sig.is_cuda
    run_dev = sig.device if sig.is_cuda else dev
    if not torch.is_tensor(J) and (isinstance(J, SupportSet) or hasattr(J, "indices")):
        Js = as_support(J)
        if Js.N != N:
            raise InvalidInputError("signal modulus does not match support")
        jt = Js.device_tensor(run_dev)
        nsup, k = 1, len(Js)
    else:
        jt = J if torch.is_tensor(J) else torch.as_tensor(np.asarray(J, dtype=np.int64))
        if jt.dim() != 2 or jt.shape[0] != B:
            raise InvalidInputError("per-signal supports must be a (B, k) tensor")
        if host_out:  # host rows: host threads derive pivots and gather, the device transforms
            jh = jt.to("cpu", dtype=torch.int64).contiguous()
            res = torch.empty((B, jh.shape[1]), dtype=sig.dtype, pin_memory=True)
            with torch.cuda.device(run_dev):
                _lib.check(_lib.load().sfft_hidft_to_dft_fused_host(
                    jh.data_ptr(), jh.shape[1], M, sig.data_ptr(), B, sig.stride(0), _DT[sig.dtype], res.data_ptr(),
                    res.shape[1], _host_threads(), _lib.stream_ptr(run_dev)))
            return res[0] if single else res
        jt = jt.to(run_dev, dtype=torch.int64, non_blocking=True).contiguous()
        nsup, k = B, jt.shape[1]
        Js = None
    code = _DT[sig.dtype]
    if out is not None:
        if single and torch.is_tensor(out) and out.dim() == 1:
            out = out.unsqueeze(0)
        _check_out(out, (B, k), sig.dtype, run_dev, "out")
    if status is not None:
        if not torch.is_tensor(status) or status.dtype != torch.int32 or status.device != run_dev \
                or status.dim() != 1 or status.numel() < nsup or status.stride(0) != 1:
            raise InvalidInputError(f"status must be a contiguous int32 tensor of >= {nsup} elements on {run_dev}")
    if out is None and not (host_out and Js is not None):
        out = torch.empty((B, k), dtype=sig.dtype, device=run_dev)
    lib = _lib.load()
    stream = _lib.stream_ptr(run_dev)
    st = status
    if Js is not None:
        # shared support: plan once (cached on J), then one gather+butterfly
        # launch per batch with the plan's tables read through L1
        cls = classify(Js)
        if not cls.is_homogeneous:
            raise ContractViolationError("hidft_to_dft requires a homogeneous support")
        plan = get_plan(Js, cls.pivots, 0, code, run_dev)
        if host_out:  # host-resident signals: host gather of the needed samples, pipelined DMA
            res = _host_transform(sig, plan, 0, _lib.OUT_DFT, k)
            return res[0] if single else res
        _lib.check(lib.sfft_hidft(plan.handle, sig.data_ptr(), B, sig.stride(0), 0, _lib.OUT_DFT,
                                  out.data_ptr(), out.stride(0), None, 0, stream))
        return out[0] if single else out
    if st is None and check:
        st = torch.zeros(nsup, dtype=torch.int32, device=run_dev)
    _lib.check(lib.sfft_hidft_to_dft_fused(jt.data_ptr(), k, nsup, M, sig.data_ptr(), B, sig.stride(0),
                                           code, out.data_ptr(), out.stride(0),
                                           st.data_ptr() if st is not None else None, stream))
    if check and st is not None:
        bad = st.cpu().numpy()
        if (bad == 2).any():
            raise InvalidInputError(f"support row {int(np.argmax(bad == 2))} is not a valid SupportSet")
        if (bad == 3).any():
            raise ContractViolationError(
                f"hidft_to_dft requires a homogeneous support (row {int(np.argmax(bad == 3))})")
    return out[0] if single else out


def hidft_to_dft_interleaved(signals, J, out=None, shift: int = 0):
    """hidft_to_dft for a batch stored sample-major: `signals` is an (N, B)
    CUDA tensor whose column b is signal b (any row stride >= B, unit column
    stride).  Returns (B, k) coefficients in ascending-J order, identical to
    hidft_to_dft_batched(signals.T.contiguous(), J); `shift` reads the
    samples at (I - shift) mod N (core.py:3-6).  The gather reads each
    needed sample index of SG neighbouring signals as one contiguous run
    (sfft_hidft_interleaved) instead of one 128 B line per sample."""
    with _device_guard(signals):
        return _hidft_to_dft_interleaved(signals, J, out, shift)


def _hidft_to_dft_interleaved(signals, J, out, shift):
    torch = _torch()
    _lib.require_device()
    if not torch.is_tensor(signals) or not signals.is_cuda or signals.dim() != 2:
        raise InvalidInputError("signals must be an (N, B) CUDA tensor")
    if signals.dtype not in (torch.complex64, torch.complex128):
        raise InvalidInputError("signals must be complex64 or complex128")
    N, B = signals.shape
    if signals.stride(1) != 1 or signals.stride(0) < B:
        raise InvalidInputError("signals need unit column stride and row stride >= B")
    Js = as_support(J)
    if Js.N != N:
        raise InvalidInputError("signal modulus does not match support")
    cls = classify(Js)
    if not cls.is_homogeneous:
        raise ContractViolationError("hidft_to_dft requires a homogeneous support")
    dev = signals.device
    plan = get_plan(Js, cls.pivots, 0, _DT[signals.dtype], dev)
    k = len(Js)
    if out is None:
        out = torch.empty((B, k), dtype=signals.dtype, device=dev)
    else:
        _check_out(out, (B, k), signals.dtype, dev, "out")
    _lib.check(_lib.load().sfft_hidft_interleaved(plan.handle, signals.data_ptr(), B, signals.stride(0), int(shift),
                                                  _lib.OUT_DFT, out.data_ptr(), out.stride(0), _lib.stream_ptr(dev)))
    return out


class stream_chain:
    """Context manager: consecutive library calls on `stream` (default: the
    current stream of the current device) may overlap through programmatic
    dependent launch (include/structfft_b200.h, sfft_stream_chain).  Inside
    the scope, no other kernel on that stream may write the inputs of a
    library call; outside any scope every call starts fully stream-ordered.
    Used by bench.py around its timed steps and captured graphs."""

    def __init__(self, stream=None):
        self._stream = stream

    def __enter__(self):
        torch = _torch()
        st = self._stream if self._stream is not None else torch.cuda.current_stream()
        self._ptr = st.cuda_stream if hasattr(st, "cuda_stream") else int(st)
        _lib.check(_lib.load().sfft_stream_chain(self._ptr, 1))
        return self

    def __exit__(self, *exc):
        _lib.load().sfft_stream_chain(self._ptr, 0)
        return False
