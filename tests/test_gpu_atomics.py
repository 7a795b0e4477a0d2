"""Device forms of the reference's _atomics primitives (test_async.py:23-91,
verify.py:368-381), called through the C ABI on device buffers."""

import numpy as np
import pytest
import torch

from paper_1707_06468_b200 import _lib

pytestmark = pytest.mark.gpu


def _st():
    return _lib.stream_ptr()


def test_gather_scatter_exchange(cuda):
    L = _lib.load()
    arr = torch.arange(5, dtype=torch.float64, device=cuda)
    idx = torch.tensor([4, 0, 2], dtype=torch.int64, device=cuda)
    out = torch.empty(3, dtype=torch.float64, device=cuda)
    _lib.check(L.ps_atomic_gather(arr.data_ptr(), 5, idx.data_ptr(), 3, out.data_ptr(), _st()))
    assert out.tolist() == [4.0, 0.0, 2.0]
    d = torch.ones(3, dtype=torch.float64, device=cuda)
    _lib.check(L.ps_atomic_scatter_add(arr.data_ptr(), 5, idx.data_ptr(), 3, d.data_ptr(), _st()))
    assert arr.tolist() == [1.0, 1.0, 3.0, 3.0, 5.0]
    val = torch.tensor([7.0], dtype=torch.float64, device=cuda)
    old = torch.empty(1, dtype=torch.float64, device=cuda)
    one = torch.tensor([1], dtype=torch.int64, device=cuda)
    _lib.check(L.ps_atomic_exchange(arr.data_ptr(), 5, one.data_ptr(), 1, val.data_ptr(), old.data_ptr(), _st()))
    assert old.item() == 1.0 and arr[1].item() == 7.0


def test_fetch_add_and_index_errors(cuda):
    L = _lib.load()
    c = torch.zeros(1, dtype=torch.int64, device=cuda)
    old = torch.empty(1, dtype=torch.int64, device=cuda)
    _lib.check(L.ps_atomic_fetch_add_i64(c.data_ptr(), 1, 0, 5, old.data_ptr(), _st()))
    assert old.item() == 0 and c.item() == 5
    with pytest.raises(IndexError):
        _lib.check(L.ps_atomic_fetch_add_i64(c.data_ptr(), 1, 3, 5, old.data_ptr(), _st()))
    arr = torch.zeros(2, dtype=torch.float64, device=cuda)
    bad = torch.tensor([9], dtype=torch.int64, device=cuda)
    d = torch.ones(1, dtype=torch.float64, device=cuda)
    with pytest.raises(IndexError):
        _lib.check(L.ps_atomic_scatter_add(arr.data_ptr(), 2, bad.data_ptr(), 1, d.data_ptr(), _st()))
    assert arr.tolist() == [0.0, 0.0]  # nothing applied when any index is bad


def test_concurrent_adds_are_exact(cuda):
    """C8: concurrent fp64 atomic adds lose nothing (8 x 1e5 in the reference;
    here 4096 device threads x 2000 adds on ONE cell)."""
    L = _lib.load()
    cell = torch.zeros(1, dtype=torch.float64, device=cuda)
    _lib.check(L.ps_atomic_add_repeat(cell.data_ptr(), 1.0, 2000, 4096, _st()))
    assert cell.item() == 4096.0 * 2000.0


def test_exchange_credit_conserves_total(cuda):
    """test_async.py:74-91: crediting against the swapped-out value never
    loses an update — exercised by many warps swapping alpha in ps_run; here
    the primitive on one cell from many threads."""
    L = _lib.load()
    arr = torch.zeros(1, dtype=torch.float64, device=cuda)
    m = 4096
    idx = torch.zeros(m, dtype=torch.int64, device=cuda)
    vals = torch.from_numpy(np.random.default_rng(0).standard_normal(m)).to(cuda)
    old = torch.empty(m, dtype=torch.float64, device=cuda)
    _lib.check(L.ps_atomic_exchange(arr.data_ptr(), 1, idx.data_ptr(), m, vals.data_ptr(), old.data_ptr(), _st()))
    total = float((vals - old).sum().item())
    assert total == pytest.approx(arr.item(), abs=1e-9)
