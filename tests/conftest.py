import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")


def pytest_collection_modifyitems(config, items):
    # Without a GPU, -m gpu tests would fail on the missing device; they are
    # selected explicitly by the driver on the B200 box.
    pass
