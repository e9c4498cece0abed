"""Runs the C++ API suite (tests/cpp/test_cpp_api.cpp): the reference's solver
test cases written against include/otdr_b200/otdr.hpp, i.e. the reference's own
C++ API names on the B200 backend."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_cpp_api")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2305_18483_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_api_host_cases():
    _build()
    out = subprocess.run([BIN, "--cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_api_device_cases():
    if not os.path.exists(BIN):
        _build()
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
