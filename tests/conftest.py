import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large CPU-oracle cases")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        j = json.load(f)
    a = np.load(os.path.join(GOLDEN, "golden.npz"))
    return j, a


@pytest.fixture(scope="session")
def port():
    import oracle

    return oracle.port()


@pytest.fixture(scope="session")
def ref():
    import oracle

    oracle.build()
    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference build) not available")
    return oracle.ref()


@pytest.fixture(scope="session")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2505_18563_b200 as pb

    return pb


@pytest.fixture(scope="session")
def cuda(pb):
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
