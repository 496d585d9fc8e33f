"""bench.py keeps the driver's contract: one JSON line with the required keys,
the roofline / e2e / clocks objects and a positive launch count."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cfg", [1, 2])
def test_bench_line_contract(cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "7", "--warmup", "3",
           "--no-cpu", "--soak", "0.2", "--e2e-steps", "3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in line, key
    assert line["steps"] == 7 and line["warmup"] == 3 and line["value"] > 0
    assert line["gpu_launches"] >= 7
    roof = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in roof, key
    assert 0 < roof["frac"] <= 1.0
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert "workload" in line["config"]
    assert line["parity"]["rel_l2_vs_planted_max"] < line["parity"]["tol"]
