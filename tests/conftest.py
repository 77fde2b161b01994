import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built extension")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture
def lib_options():
    """Set library dispatch options (lfmmi_set_option) for one test; every
    option is reset to its default afterwards."""
    from paper_2005_09824_b200 import _backend

    e = _backend.ext()

    def set_(**kw):
        for k, v in kw.items():
            e.set_option(k, str(v))

    yield set_
    e.reset_options()
