"""Same error behaviour as the reference: every case of
tests/golden/error_cases.json (outcomes recorded from the unmodified
reference by tests/golden/make_golden_errors.py) gives the same outcome --
"ok" or the same exception class -- through the device package."""

import json
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from make_golden_errors import run_case  # noqa: E402

CASES = json.load(open(os.path.join(HERE, "golden", "error_cases.json")))


@pytest.fixture(scope="module")
def S():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2211_15299_b200 as S
    return S


@pytest.mark.parametrize("case", CASES, ids=[f"{i}-{c['op']}" for i, c in enumerate(CASES)])
def test_same_outcome_as_reference(S, case):
    assert run_case(S, case) == case["expect"], case
