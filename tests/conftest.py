"""Shared pytest setup: the `gpu` marker and import paths.

`-m "not gpu"` runs the oracle KATs, host logic and ABI-load checks on CPU;
`-m gpu` runs the parity suite on a B200 through the C-ABI library.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def ora():
    import pyoracle

    pyoracle.lib()
    return pyoracle
