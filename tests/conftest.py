import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden_hidft():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_hidft.npz"))


@pytest.fixture(scope="session")
def golden_configs():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_configs.npz"))


@pytest.fixture(scope="session")
def kats():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "kats.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_sas():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden_sas.npz"))


@pytest.fixture(scope="session")
def plan_digests():
    """sha256 digests of the unmodified reference's plan tables at the BASELINE
    config sizes (tests/golden/make_golden_plan_digests.py)."""
    import json
    with open(os.path.join(ROOT, "tests", "golden", "plan_digests.json")) as fh:
        return json.load(fh)


def table_digest(a, dt):
    import hashlib
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a).astype(dt)).tobytes()).hexdigest()


def twiddle_sample_index(n):
    """The positions make_golden_plan_digests.py sampled from a table of n twiddles."""
    import numpy as np
    if n <= 512:
        return np.arange(n, dtype=np.int64)
    return np.unique(np.concatenate([np.arange(64), (np.arange(448) * 2654435761 % n)])).astype(np.int64)
