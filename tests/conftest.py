"""Test configuration.

`-m "not gpu"` runs here on CPU: the oracle against the reference's golden
vectors, host-side logic, the C-ABI export check and world_size-2 gloo tests.
`-m gpu` needs a B200: parity of the sm_100a path against the oracle.
"""

import os
import sys

# before anything initialises CUDA (see paper_1908_04207_b200/__init__.py)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")
    # in-round device watchdog for tests: fail fast instead of hanging a box
    os.environ.setdefault("EC_TIMEOUT_S", "20")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "multigpu" in item.keywords:
            item.add_marker(pytest.mark.gpu)


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def need_gpus(n: int):
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} CUDA device(s)")
