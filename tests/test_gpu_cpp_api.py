"""The C++ drop-in surface (include/pdsim/*.hpp over libpdsim_gpu.so) passes
the reference's own sim_engine_test cases restated in tests/native/cpp_api_test.cpp."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_api_program():
    exe = os.path.join(ROOT, "tests", "native", "cpp_api_test")
    assert os.path.exists(exe), "run `make` (or __graft_entry__.build()) first"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp_api_test: ok" in r.stdout
