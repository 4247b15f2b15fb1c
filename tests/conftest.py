import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through liblffn_gpu.so)")


def _ensure_built():
    # The checkers are test infrastructure; build them on demand.  The
    # reference build needs /root/reference (this container only); on the GPU
    # box the prebuilt oracle/_ref/liblffn_ref.so travels with the snapshot.
    so = os.path.join(ROOT, "oracle", "liblffn_oracle.so")
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), so], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "liblffn_ref.so")
    if not os.path.exists(ref) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    lib = os.path.join(ROOT, "paper_2403_07221_b200", "csrc", "liblffn_gpu.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2403_07221_b200", "csrc")],
                       check=True)
    dropin = os.path.join(ROOT, "oracle", "_ref", "dropin_test")
    if not os.path.exists(dropin) and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True)


_ensure_built()

if os.environ.get("LFFN_TEST_CHECKED"):
    # run the suite against the bounds-checked build (device asserts on
    # data-derived indices; compute-sanitizer is closed on the GPU pool)
    from paper_2403_07221_b200 import _capi as _c

    _c.LIB_PATH = os.path.join(ROOT, "paper_2403_07221_b200", "csrc", "liblffn_gpu_checked.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("reference build (oracle/_ref) unavailable")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda:0")
