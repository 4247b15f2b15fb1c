"""The reference's forward-path checks, compiled against the reference's own
headers/sources and re-pointed at the GPU through the C++ drop-in
(include/lffn_gpu_dropin.hpp) -- oracle/dropin_test.cpp."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_test")


def test_reference_checks_through_cpp_dropin():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: build it with `make -C oracle dropin` where /root/reference exists")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK (0 failures)" in r.stdout
