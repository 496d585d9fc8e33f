"""Sharded batch with the result rows gathered through peer memory
(dist.PeerRows): two processes (gloo for the host-side
plumbing) each transform their row shard and write it straight into rank 0's
device buffer via CUDA IPC.  The box gives one GPU, so both processes map
the same device; on a node the ranks sit on different GPUs and the same
stores travel over NVLink / NVSwitch.  The ranks never wait on each other's
kernels: each synchronises its own stream, then a barrier."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, B, q):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch
    import torch.distributed as dist
    try:
        import paper_2211_15299_b200 as S
        from paper_2211_15299_b200 import workloads as W
        from paper_2211_15299_b200.dist import PeerRows, shard_range
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        a, b = shard_range(B, rank, world)
        wl = W.make_workload(cfg, B=b - a, b0=a)
        dt = torch.complex64 if wl.dtype == "complex64" else torch.complex128
        sig = torch.empty((b - a, wl.N), dtype=dt, device="cuda")
        W.synthesize_into(sig, wl.support, wl.coeffs)
        peer = PeerRows(B, wl.k, dt)
        assert peer.rows == (a, b)
        J = S.SupportSet(wl.N, wl.support) if wl.support.ndim == 1 else torch.from_numpy(wl.support).cuda()
        S.hidft_to_dft_batched(sig, J, out=peer.local)
        full = peer.complete()
        res = True
        if rank == 0:
            want = W.make_workload(cfg, B=B).coeffs
            got = full.cpu().numpy()
            err = np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)
            res = float(err.max())
        peer.close()
        q.put((rank, res))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("cfg,B", [(2, 24), (4, 21), (1, 16)])
def test_peer_rows_world2(cfg, B):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[1] is True, res[1]
    tol = 1e-5 if cfg != 1 else 1e-11
    assert isinstance(res[0], float) and res[0] < tol, res[0]
