"""Runs the C++ drop-in test (tests/cpp/test_dropin.cpp, prebuilt into
oracle/_ref/test_dropin in the build container): the reference's own types and
functions against include/diloco_cuda.hpp on the GPU, bitwise."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "test_dropin")


def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    if p.returncode == 2:
        pytest.skip("no CUDA device")
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    assert "0 failed" in p.stdout
