import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: CPU test taking more than ~20 s")


import pytest  # noqa: E402


@pytest.fixture(autouse=True)
def _release_device_memory():
    """Full-size tests need most of the 180 GB: hand the caching allocator's
    blocks back after every GPU test."""
    yield
    try:
        import torch
        if torch.cuda.is_available():
            import gc
            gc.collect()
            torch.cuda.empty_cache()
    except ImportError:
        pass
