import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA product path")
    config.addinivalue_line("markers", "slow: long-running CPU checks")


def has_reference():
    from pyoracle import REF_SO
    return os.path.exists(REF_SO)


requires_reference = pytest.mark.skipif(not has_reference(), reason="oracle/_ref/libbtref.so not built")
