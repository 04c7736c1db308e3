import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    # `-m gpu` tests are never skipped: on a box without a working B200 they fail
    # loudly, because they are the product's correctness gate.
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI CUDA path)")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
