"""CPU-only tests: C-ABI library loading/exports, host-side validation,
workload generators vs the reference's golden supports, sharding logic,
and the multi-process gather over gloo (world_size 2)."""

import hashlib
import os
import re
import socket

import numpy as np
import pytest

import structfft_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "structfft_b200.h")) as fh:
        text = fh.read()
    return re.findall(r"SFFT_API\s+[\w\s\*]+?\b(sfft_\w+)\s*\(", text)


def test_library_exports_every_header_symbol():
    from paper_2211_15299_b200 import _lib
    lib = _lib.load()
    names = header_symbols()
    assert len(names) >= 13
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert bound == set(names)
    assert lib.sfft_version().startswith(b"structfft_b200")


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2211_15299_b200", "libsfft_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def test_support_set_validation():
    from paper_2211_15299_b200 import InvalidInputError, SupportSet
    with pytest.raises(InvalidInputError):
        SupportSet.make(12, [0])
    with pytest.raises(InvalidInputError):
        SupportSet.make(8, [])
    with pytest.raises(InvalidInputError):
        SupportSet.make(8, [8])
    with pytest.raises(InvalidInputError):
        SupportSet.make(8, [1, 1])
    with pytest.raises(InvalidInputError):
        SupportSet(8, [3, 1])
    J = SupportSet.make(32, [27, 3, 17, 25])
    assert J.indices == (3, 17, 25, 27)
    assert J.M == 5 and len(J) == 4 and 17 in J and 18 not in J
    assert J == SupportSet(32, [3, 17, 25, 27]) and hash(J) == hash(SupportSet(32, (3, 17, 25, 27)))
    with pytest.raises(AttributeError):
        J.N = 64


def test_pivot_vector_validation():
    from paper_2211_15299_b200 import InvalidInputError, validate_pivot_vector, v2
    assert validate_pivot_vector([0, 2, 5], 10) == (0, 2, 5)
    with pytest.raises(InvalidInputError):
        validate_pivot_vector([2, 1], 10)
    with pytest.raises(InvalidInputError):
        validate_pivot_vector([10], 10)
    assert v2(12) == 2 and v2(-8) == 3
    with pytest.raises(InvalidInputError):
        v2(0)


def test_compute_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2211_15299_b200 as S
    J = S.SupportSet.make(32, [3, 17, 25, 27])
    with pytest.raises(S.DeviceError):
        S.pivots(J)
    with pytest.raises(S.DeviceError):
        S.hidft(np.zeros(32, complex), J, (1, 3))
    with pytest.raises(S.DeviceError):
        S.hidft_to_dft_batched(np.zeros((2, 32), np.complex64), J)


def test_workload_supports_match_reference(golden_configs):
    from paper_2211_15299_b200 import workloads as W
    g = golden_configs
    for c in (1, 2, 3, 5):
        J, M = W.config_support(c)
        assert np.array_equal(J, g[f"cfg{c}_J"])
    h = hashlib.sha256()
    for b in range(256):
        J, _ = W.config_support(4, b)
        if b < 8:
            assert np.array_equal(J, g[f"cfg4_J{b}"])
        h.update(J.astype("<i8").tobytes())
    assert h.digest() == bytes(g["cfg4_sha256_first256"])
    for c in (1, 2, 3, 4):
        wl = W.make_workload(c, 2)
        for b in range(2):
            np.testing.assert_array_equal(wl.coeffs[b], g[f"cfg{c}_b{b}_coef"])


def test_shard_range():
    from paper_2211_15299_b200.dist import shard_range
    for B in (0, 1, 7, 16, 1024, 8193):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, B, k, q):
    import torch
    import torch.distributed as dist
    from paper_2211_15299_b200.dist import gather_rows, shard_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    full = torch.arange(B * k, dtype=torch.float64).reshape(B, k)
    full = torch.complex(full, -full)
    try:
        a, b = shard_range(B, rank, world)
        got = gather_rows(full[a:b].clone(), B)
        q.put((rank, bool(torch.equal(got, full))))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [16, 13])
def test_gather_rows_gloo_world2(B):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, B, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_oracle_reference_call_on_workload():
    from paper_2211_15299_b200 import workloads as W
    wl = W.make_workload(1, 2)
    f = O.synthesize(wl.support, wl.coeffs[0], wl.M)
    got = O.reference_call(f, wl.support, wl.M)
    assert np.linalg.norm(got - wl.coeffs[0]) / np.linalg.norm(wl.coeffs[0]) < 1e-12


def test_capi_demo_compiles_with_plain_c(tmp_path):
    """The C-ABI is usable from plain C (gcc, no torch): compile and link the demo."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    exe = tmp_path / "capi_demo"
    cmd = ["gcc", "-O2", os.path.join(ROOT, "examples", "capi_demo.c"), "-I", os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", "-L", os.path.join(ROOT, "paper_2211_15299_b200"), "-lsfft_b200",
           "-L/usr/local/cuda/lib64", "-lcudart", "-lm", "-o", str(exe)]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the driver's reference arm) runs on the
    host alone: one JSON line with the contract's keys from rank 0, nothing
    from the other ranks."""
    import json
    import subprocess
    import sys
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1", "--steps", "2",
           "--warmup", "3", "--ref-seconds", "10"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    want_kind = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "structfft")) else "port"
    assert line["cpu_baseline"]["kind"] == want_kind and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    other = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert other.returncode == 0 and other.stdout.strip() == ""


def test_bench_gpus_flag_relaunches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks
    (torch.distributed.run on 127.0.0.1): exactly one JSON line, from rank 0,
    reporting n_gpus = 2.  Run on the reference arm, which needs no GPU."""
    import json
    import subprocess
    import sys
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--config", "1",
           "--steps", "1", "--warmup", "3", "--ref-seconds", "5"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "batch shard x2"
    assert line["config"]["global_batch"] == 2 * 16


def test_bench_gpus_mismatch_and_no_device_fail_loudly():
    """--gpus that disagrees with WORLD_SIZE is refused; the b200 arm without
    a CUDA device exits non-zero instead of falling back to the CPU."""
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "1", "--no-per-config"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0
