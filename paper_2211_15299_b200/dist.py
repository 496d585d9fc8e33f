"""Batch sharding over GPUs.

Signals are independent: rank g owns the contiguous slice
[g*B/G, (g+1)*B/G) of the batch (and of the per-signal supports), with no
data-path collective.  The only exchange is the optional final gather of
the B x k coefficients: either one all_gather over NCCL (NVLink / NVSwitch
on a B200 node; gloo in the CPU tests), or, with PeerRows, no collective at
all: each rank's transform writes its rows straight into the owner's device
buffer through CUDA IPC peer memory.
"""

from __future__ import annotations


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of B items for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(B, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local, B: int, group=None):
    """All-gather row shards (each rank's contiguous slice) into (B, ...)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(B, r, world) for r in range(world)]
    width = max(b - a for a, b in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    if local.is_complex():
        pad = torch.view_as_real(pad)
    buf = torch.empty((world * width,) + tuple(pad.shape[1:]), dtype=pad.dtype, device=pad.device)
    dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
    buf = buf.view((world, width) + tuple(pad.shape[1:]))
    if local.is_complex():
        buf = torch.view_as_complex(buf)
    return torch.cat([buf[r, : b - a] for r, (a, b) in enumerate(sizes)], dim=0)


def _lib_error(_lib, what):
    from .errors import DeviceError
    detail = _lib.load().sfft_last_error().decode(errors="replace")
    return DeviceError(f"{what}: {detail}" if detail else what)


class _DeviceArray:
    """__cuda_array_interface__ view of raw device memory (zero-copy into torch)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "strides": None, "version": 3}


class PeerRows:
    """A (B, width) result buffer on rank `owner`'s GPU that every rank of
    the group writes its row shard into directly.

    The owner allocates it (sfft_peer_alloc) and broadcasts the CUDA IPC
    handle; the other ranks map it (sfft_peer_open).  `local` is this rank's
    rows [shard_range(B, rank, world)) of the mapped buffer: pass it as the
    `out` of hidft_to_dft_batched and the transform's epilogue stores go over
    NVLink / NVSwitch to the owner.  After every rank has synchronised its
    stream and the group has passed a barrier (`complete()`), `full` on the
    owner holds all B rows.  Processes sharing one GPU use the same path
    (IPC within a device), which is how the tests exercise it."""

    def __init__(self, B: int, width: int, dtype, group=None, owner: int = 0):
        import ctypes

        import torch
        import torch.distributed as dist

        from . import _lib
        self._dist, self._group, self.owner = dist, group, owner
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.B, self.width, self.dtype = B, width, dtype
        esz = {torch.complex64: 8, torch.complex128: 16}[dtype]
        typestr = {torch.complex64: "<c8", torch.complex128: "<c16"}[dtype]
        lib = _lib.load()
        self._lib, self._ptr = lib, ctypes.c_void_p()
        dev = torch.device("cuda", torch.cuda.current_device())
        # every rank takes the same path through the collectives, even when
        # the allocation or a mapping fails (then all ranks raise together)
        msg = [None]
        if self.rank == owner:
            handle = (ctypes.c_ubyte * _lib.IPC_HANDLE_BYTES)()
            if lib.sfft_peer_alloc(max(1, B * width * esz), ctypes.byref(self._ptr), handle) == _lib.OK:
                msg = [bytes(handle)]
        dist.broadcast_object_list(msg, src=dist.get_global_rank(group, owner) if group is not None else owner,
                                   group=group)
        if msg[0] is None:
            raise _lib_error(_lib, "peer buffer allocation failed on the owner rank")
        opened = True
        if self.rank != owner:
            handle = (ctypes.c_ubyte * _lib.IPC_HANDLE_BYTES).from_buffer_copy(msg[0])
            opened = lib.sfft_peer_open(handle, ctypes.byref(self._ptr)) == _lib.OK
        flag = torch.tensor([1 if opened else 0], dtype=torch.int32,
                            device=dev if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag.item()) == 0:
            if not opened:
                self._ptr = ctypes.c_void_p()
            self.local = self.full = None
            self.close()
            raise _lib_error(_lib, "a rank could not map the owner's result buffer (CUDA IPC / peer access)")
        base = int(self._ptr.value)
        a, b = shard_range(B, self.rank, self.world)
        self.rows = (a, b)
        self.local = torch.as_tensor(_DeviceArray(base + a * width * esz, (b - a, width), typestr), device=dev)
        self.full = (torch.as_tensor(_DeviceArray(base, (B, width), typestr), device=dev)
                     if self.rank == owner else None)

    def complete(self):
        """Every rank's stores are done: sync this rank's device, then barrier."""
        import torch
        torch.cuda.synchronize()
        self._dist.barrier(group=self._group)
        return self.full

    def close(self):
        """Unmap (other ranks) before the owner frees the buffer.  Collective:
        every rank calls it once."""
        if getattr(self, "_closed", False):
            return
        self._closed = True
        self.local = self.full = None
        if self.rank != self.owner and self._ptr.value is not None:
            self._lib.sfft_peer_close(self._ptr)
        self._dist.barrier(group=self._group)
        if self.rank == self.owner and self._ptr.value is not None:
            self._lib.sfft_peer_free(self._ptr)
        self._ptr = type(self._ptr)()
