"""Opt-in experimental kernels (selected by environment variables read once
per process, so each runs in its own subprocess) produce the same y as the
default path: the shared-memory-staged gather (LFFN_GATHER_ASYNC) and the
warp-specialised fused kernel with staged gather warps (LFFN_FUSED_ASYNC)
walk the same records in the same table order -- bit-identical."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "path_ab_check.py")


def _run(tmp_path, tag, env, extra=()):
    out = str(tmp_path / tag)
    subprocess.run([sys.executable, TOOL, "c2", "4096", out, *extra], check=True,
                   env={**os.environ, **env}, timeout=600)
    return np.load(out + ".npy")


@pytest.mark.parametrize("variant", [
    ("gather_async", {"LFFN_GATHER_ASYNC": "1,3,16"}, ()),
    ("fused_async", {"LFFN_FUSED_ASYNC": "16,3", "LFFN_FUSED_MIN_TOKENS": "1"}, ("--fused",)),
    ("fused_regs", {"LFFN_FUSED_MIN_TOKENS": "1"}, ("--fused",)),
], ids=lambda v: v[0])
def test_experimental_paths_bit_identical(tmp_path, variant):
    tag, env, extra = variant
    base = _run(tmp_path, "base", {})
    alt = _run(tmp_path, tag, env, extra)
    assert np.array_equal(base, alt)
