"""Runs the C++ drop-in test binary (tests/cpp/test_dropin.cpp, built by
`make -C oracle dropin` where the reference sources exist): the reference's
own types, fixtures and CPU functions checked against weft::gpu::*."""
import os
import subprocess

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.ref]
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "test_dropin")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_dropin not built")
def test_cpp_dropin():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout
