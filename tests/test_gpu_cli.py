"""CLI parity: our `transform` / `analyze` against the reference CLI's outputs
(tests/golden/make_golden_cli.py) on the same JSON inputs."""

import glob
import io
import json
import os
from contextlib import redirect_stdout

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _close(a, b, path=""):
    if isinstance(a, dict):
        assert set(a) == set(b), path
        for k in a:
            _close(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _close(x, y, f"{path}[{i}]")
    elif isinstance(a, float) or isinstance(b, float):
        assert abs(a - b) <= 1e-9 * max(1.0, abs(b)), (path, a, b)
    else:
        assert a == b, (path, a, b)


@pytest.mark.parametrize("ref_file", sorted(glob.glob(os.path.join(HERE, "ref_*.json"))),
                         ids=lambda p: os.path.basename(p))
def test_cli_matches_reference(ref_file):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_15299_b200 import cli
    ref = json.load(open(ref_file))
    argv = [a.replace("{DIR}", HERE) for a in ref["argv"]]
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == ref["rc"]
    got, want = json.loads(buf.getvalue()), json.loads(ref["stdout"])
    if argv[0] == "analyze":
        got.pop("doubling"), want.pop("doubling")  # sumset statistic: out of scope
    _close(got, want)


def test_cli_exit_codes(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_15299_b200 import cli
    assert cli.main(["transform", "--signal", str(tmp_path / "missing.json"), "--algo", "hidft"]) == 2
    bad = tmp_path / "generic.json"
    bad.write_text(json.dumps({"N": 64, "support": [3, 17, 25, 27, 35], "coeffs": [[1, 0]] * 5}))
    assert cli.main(["transform", "--signal", str(bad), "--algo", "hidft"]) == 3
