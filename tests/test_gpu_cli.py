"""CLI parity: our `structfft` commands against the reference CLI's outputs
(tests/golden/make_golden_cli.py) on the same JSON inputs: analyze (binary,
ascii / dot trees, doubling), transform with every --algo, gen for every
family kind (the support and signal files byte-identical), bench on a
scenario file (operation counts and supports identical; errors within
tolerance)."""

import csv
import glob
import io
import json
import os
from contextlib import redirect_stdout

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
LOOSE = {"max_rel_err", "ops_over_klogk_mean"}  # float statistics of the decoded values


def _close(a, b, path="", tol=1e-9):
    if isinstance(a, dict):
        assert set(a) == set(b), path
        for k in a:
            _close(a[k], b[k], f"{path}.{k}", tol)
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _close(x, y, f"{path}[{i}]", tol)
    elif isinstance(a, float) or isinstance(b, float):
        key = path.rsplit(".", 1)[-1]
        if key in LOOSE:
            assert a <= 1e-8 and b <= 1e-8 if key == "max_rel_err" else abs(a - b) <= 1e-6 * abs(b), (path, a, b)
        else:
            assert abs(a - b) <= tol * max(1.0, abs(b)), (path, a, b)
    else:
        assert a == b, (path, a, b)


@pytest.mark.parametrize("ref_file", sorted(glob.glob(os.path.join(HERE, "ref_*.json"))),
                         ids=lambda p: os.path.basename(p))
def test_cli_matches_reference(ref_file, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_15299_b200 import cli
    ref = json.load(open(ref_file))
    argv = [a.replace("{DIR}", HERE).replace("{OUT}", str(tmp_path)) for a in ref["argv"]]
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = cli.main(argv)
    assert rc == ref["rc"]
    got, want = json.loads(buf.getvalue().replace(str(tmp_path), "{OUT}")), json.loads(ref["stdout"])
    # submatrix solves the k x k Vandermonde in the conjugate orientation (samples f(-j),
    # nodes e^{-2 pi i l/N}) on the device: same system, rounding of its conditioning
    tol = 1e-6 if "submatrix" in ref_file else 1e-9
    _close(got, want, tol=tol)
    for name, content in ref["files"].items():
        path = os.path.join(str(tmp_path), name)
        assert os.path.exists(path), name
        if name.endswith(".csv"):
            rows_g = list(csv.reader(open(path)))
            rows_w = list(csv.reader(io.StringIO(content)))
            assert rows_g[0] == rows_w[0] and len(rows_g) == len(rows_w)
            ci = rows_w[0].index("max_rel_err")
            for rg, rw in zip(rows_g[1:], rows_w[1:]):
                assert rg[:ci] == rw[:ci], (rg, rw)  # supports, plans and exact op counts
                assert float(rg[ci]) <= 1e-8 and float(rw[ci]) <= 1e-8
        else:
            assert open(path).read() == content, name


def test_cli_exit_codes(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2211_15299_b200 import cli
    assert cli.main(["transform", "--signal", str(tmp_path / "missing.json"), "--algo", "hidft"]) == 2
    bad = tmp_path / "generic.json"
    bad.write_text(json.dumps({"N": 64, "support": [3, 17, 25, 27, 35], "coeffs": [[1, 0]] * 5}))
    assert cli.main(["transform", "--signal", str(bad), "--algo", "hidft"]) == 3
    big = tmp_path / "big.json"
    big.write_text(json.dumps({"N": 1 << 13, "support": [1, 2], "coeffs": [[1, 0]] * 2}))
    assert cli.main(["transform", "--signal", str(big), "--algo", "oracle"]) == 4
    assert cli.main(["gen", "--kind", "nosuch", "--params", "{}", "--out", str(tmp_path / "x.json")]) == 2
