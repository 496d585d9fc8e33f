"""The plain-C consumer of the C-ABI runs on the GPU (examples/capi_demo.c)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_capi_demo_runs(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = tmp_path / "capi_demo"
    lib = os.path.join(ROOT, "paper_2211_15299_b200")
    cmd = ["gcc", "-O2", os.path.join(ROOT, "examples", "capi_demo.c"), "-I", os.path.join(ROOT, "include"),
           "-I/usr/local/cuda/include", "-L", lib, "-lsfft_b200", "-L/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{lib}", "-o", str(exe)]
    assert subprocess.run(cmd, capture_output=True).returncode == 0
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "status 3" in out.stdout


@pytest.mark.gpu
def test_fma_peak_probe_reports_plausible_throughput():
    """sfft_probe_fma_peak (the flop-roofline denominator bench.py measures in
    its own run): fp32 and fp64 FMA throughput in the range of a B200's
    non-tensor pipes, fp32 above fp64, bad arguments rejected."""
    import ctypes
    from paper_2211_15299_b200 import _lib
    lib = _lib.load()
    got = []
    for code in (0, 1):
        v = ctypes.c_double(0.0)
        assert lib.sfft_probe_fma_peak(code, ctypes.byref(v), _lib.stream_ptr()) == 0
        got.append(v.value)
    assert 20.0 < got[0] < 100.0 and 8.0 < got[1] < 60.0 and got[0] > got[1], got
    assert lib.sfft_probe_fma_peak(7, ctypes.byref(ctypes.c_double()), None) != 0
