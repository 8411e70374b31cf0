import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def port():
    """oracle/sw_oracle.c -- the CPU restatement (checker only)."""
    from oracle import pyoracle
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference behind oracle/ref_shim.cpp; skipped where it cannot be had."""
    from oracle import pyoracle
    if not pyoracle.Ref.available():
        pytest.skip("oracle/_ref/libswref.so not present and /root/reference absent")
    return pyoracle.Ref()


@pytest.fixture(scope="session")
def b62():
    from paper_2203_11100_b200 import synth
    return synth.blosum62()


@pytest.fixture(scope="session")
def lib():
    """libswb200.so, built on demand (nvcc cross-compiles without a GPU)."""
    from paper_2203_11100_b200 import _cabi, build
    build.build_library()
    return _cabi.load()
