"""The C++ drop-in (include/flowbb_b200/gpu_backend.hpp) driving the UNMODIFIED reference
API: tests/cpp/test_dropin.cpp, compiled against the reference headers into
oracle/_ref/dropin_test by build() (where /root/reference exists) and run on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_reference_api_with_gpu_backend():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (reference sources absent at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
