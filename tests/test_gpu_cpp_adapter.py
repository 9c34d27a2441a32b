"""Runs the C++ adapter test binary (tests/cpp/test_adapter.cpp): the
reference's own unit-test expectations against include/mgcuda.hpp on the
B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_adapter_reference_cases():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_adapter")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
