"""The host->device input pipeline (pipeline.BatchPrefetcher): the device batches equal
the host source, and a planned-step run fed by it is bitwise the run fed by device
batches (the overlap only moves the copies)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_25976_b200 as P  # noqa: E402
from paper_2603_25976_b200.pipeline import BatchPrefetcher  # noqa: E402
from oracle import curvopt_oracle as O  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def _host_batches(n, b=256, n0=784, c=10):
    return [O.synthetic_batch(b, n0, c, seed=1 + i) for i in range(n)]


def test_prefetched_batches_equal_host_source():
    hb = _host_batches(5)
    pf = BatchPrefetcher(iter(hb), "ce")
    for X, y in hb[:4]:  # (the fifth is in flight when the source runs dry)
        b = pf.next()
        assert torch.equal(b.inputs.cpu(), torch.from_numpy(X.astype(np.float32)))
        assert torch.equal(b.targets.cpu(), torch.from_numpy(y.astype(np.int64)))


def test_step_run_through_prefetcher_is_bitwise_identical():
    hb = _host_batches(7)
    m = P.Model(784, (128,), 10, "relu")
    meth = P.make("sgn_ce", m)
    w0 = P.init_params(m, P.Rng(0)).to_device()
    pf = BatchPrefetcher(iter(hb), "ce")
    wa, sa = w0, meth.init(w0, 0)
    wb, sb = w0, meth.init(w0, 0)
    for X, y in hb[:6]:
        wa, sa, ia = meth.step(wa, pf.next(), sa)
        bd = P.Batch(torch.from_numpy(X.astype(np.float32)).cuda(), torch.from_numpy(y).cuda(), "ce")
        wb, sb, ib = meth.step(wb, bd, sb)
        ra, rb = np.array(ia.to_row()), np.array(ib.to_row())
        assert np.array_equal(np.isnan(ra), np.isnan(rb)) and np.array_equal(ra[~np.isnan(ra)], rb[~np.isnan(rb)])
    assert torch.equal(wa.data, wb.data)
