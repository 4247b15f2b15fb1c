"""Table shards built without the whole stack (multi-GPU table sharding).

``lffn_fill_gaussian_slice`` must return exactly elements [skip, skip + n) of
the reference's make_rng(seed) + fill_gaussian stream (common.hpp:44-49,
one distribution object over the whole stream), so a rank can build its
slice of BASELINE c4's 4.3 GB float64 stack alone; the upload of that slice
must equal the upload of the full stack restricted to the shard.
"""
import numpy as np
import pytest

from paper_2403_07221_b200 import fill_gaussian, fill_gaussian_slice
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_table_slice


@pytest.mark.parametrize("skip,n", [(0, 10), (1, 7), (501, 300), (4096, 1), (999, 0)])
def test_slice_equals_stream(skip, n):
    full = fill_gaussian(2, skip + n + 3, 0.02)
    np.testing.assert_array_equal(fill_gaussian_slice(2, skip, n, 0.02), full[skip:skip + n])


def test_slice_matches_reference_stream(reference):
    """Pinned to the reference library's own draws (oracle/_ref)."""
    full = reference.gaussian(2, 5000, 0.02)
    np.testing.assert_array_equal(fill_gaussian_slice(2, 1234, 3000, 0.02), full[1234:4234])


def test_table_slice_of_a_workload():
    w = WORKLOADS["c1"]
    _, _, T = make_params(w)
    per = (1 << w.tau) * w.d
    for kb, ke in [(0, 8), (3, 7), (7, 8), (4, 4)]:
        s = make_table_slice(w, kb, ke)
        assert s.table_range == (kb, ke)
        np.testing.assert_array_equal(s.data, T.data[kb * per:ke * per])


@pytest.mark.gpu
def test_slice_upload_equals_full_upload():
    import torch

    from paper_2403_07221_b200 import LookupFFN
    from paper_2403_07221_b200.configs import make_x

    w = WORKLOADS["c2_bf16"]
    cfg, proj, T = make_params(w)
    x = torch.from_numpy(make_x(w, 300)).cuda()
    kb, ke = 37, 101
    a = LookupFFN(cfg, proj, T, max_tokens=300, table_dtype="bf16", table_range=(kb, ke))
    b = LookupFFN(cfg, proj, make_table_slice(w, kb, ke), max_tokens=300, table_dtype="bf16",
                  table_range=(kb, ke))
    ya, yb = a.forward_device(x), b.forward_device(x)
    a.sync()
    b.sync()
    assert torch.equal(ya, yb)
    with pytest.raises(Exception):
        LookupFFN(cfg, proj, make_table_slice(w, kb, ke + 1), max_tokens=300,
                  table_range=(kb, ke))
