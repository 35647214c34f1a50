"""GPU: run the C++ drop-in layer's test program (tests/cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_dctfilter_b200")


def test_cpp_dropin(cuda):
    assert os.path.exists(BIN), "build with `make cpp-test`"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
