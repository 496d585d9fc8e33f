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
