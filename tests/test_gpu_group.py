"""The C-ABI table-sharded forward (lffn_group / lffn_forward_sharded, NCCL
owned by the group) on a world-1 communicator: every combine mode equals the
plain forward up to fp32 reassociation and the oracle within the bar.  The
multi-rank record exchange and chunk layout follow sharded.py, whose logic is
covered over gloo at world 2 and 3 (tests/test_sharded.py)."""
import numpy as np
import pytest

from gpu_helpers import assert_close, device_forward, stored_tables, to_oracle
from paper_2403_07221_b200 import LookupFFN, UsageError
from paper_2403_07221_b200.configs import WORKLOADS, make_params, make_x
from paper_2403_07221_b200.sharded import NativeTableShard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n", [("c1", 512), ("c2", 1024), ("c3", 2048)])
@pytest.mark.parametrize("chunks", [1, 4])
def test_native_group_world1(oracle, name, n, chunks):
    import torch

    w = WORKLOADS[name]
    cfg, proj, T = make_params(w)
    x = make_x(w, n)
    plain = device_forward(LookupFFN(cfg, proj, T, max_tokens=n, table_dtype=w.table_dtype), x)
    g = NativeTableShard(cfg, proj, T, rank=0, world=1, nccl_id=NativeTableShard.unique_id(),
                         max_tokens=n, table_dtype=w.table_dtype, chunks=chunks)
    xd = torch.from_numpy(x).cuda()
    scale = np.abs(plain).max()
    for combine in ("reduce_scatter", "all_reduce", "none"):
        y = g.forward(xd, combine=combine).cpu().numpy()
        assert y.shape == plain.shape
        assert np.abs(y - plain).max() <= 1e-6 * scale, combine
    c, s = to_oracle(cfg, proj)
    y_ref = oracle.lookup_forward(c, s, proj.blob, stored_tables(T.data, w.table_dtype),
                                  x.astype(np.float64))
    assert_close(y, y_ref, 1e-5, f"{name} sharded vs oracle")
    if chunks > 1:  # reduce-scatter needs n a multiple of world * chunks
        with pytest.raises(UsageError):
            g.forward(xd[: n - 1], combine="reduce_scatter")
    g.close()


def test_native_group_rejects_bad_arguments():
    w = WORKLOADS["c1"]
    cfg, proj, T = make_params(w)
    with pytest.raises(UsageError):
        NativeTableShard(cfg, proj, T, rank=1, world=1, nccl_id=b"\0" * 128, max_tokens=8)
