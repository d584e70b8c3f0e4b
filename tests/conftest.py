import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_NPZ = os.path.join(REPO, "tests", "golden", "golden.npz")
GOLDEN_JSON = os.path.join(REPO, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libkpm.so")
    config.addinivalue_line("markers", "slow: config-scale case (minutes)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_NPZ) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="session")
def golden_meta():
    import json
    with open(GOLDEN_JSON) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import netdos_oracle as orc
    orc.lib()
    return orc


GRAPH_CASES = ["triangle", "path3", "star4", "grid4x5", "isolated9", "er200", "ba300",
               "ba_p64"]


@pytest.fixture(scope="session")
def kpm_ctx():
    """The libkpm context on cuda:0 (GPU tests only)."""
    from paper_1905_09758_b200 import _lib
    return _lib.Context.get(0)
