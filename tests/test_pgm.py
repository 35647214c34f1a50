"""CPU: PGM I/O of the C++ drop-in layer (tests/cpp/test_pgm.cc)."""
import os
import subprocess

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_pgm")


def test_pgm_io():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "ALL PASSED" in r.stdout, r.stdout + r.stderr
