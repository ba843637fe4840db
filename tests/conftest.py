import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgg.so")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_small():
    with open(os.path.join(GOLDEN, "reference_small.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_rmat12():
    with open(os.path.join(GOLDEN, "rmat12.json")) as fh:
        return json.load(fh)


@pytest.fixture(autouse=True)
def _gpu_gate(request):
    if request.node.get_closest_marker("gpu") and not has_gpu():
        pytest.fail("GPU test selected but no CUDA device is visible")
