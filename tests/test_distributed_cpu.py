"""World-size-2 gloo test (CPU) of the batch-sharding algebra the native library
implements for N GPUs: every rank linearizes its b/N rows with the GLOBAL batch
size in the mean, and the gradient, loss and every curvature product are
sum-all-reduced.  The oracle plays the per-rank device; the result must equal the
single-process full-batch oracle.  Also checks bench.py's shard layout."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DIMS = (20, 16, 12, 5)
B = 24


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    from oracle import curvopt_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = O.init_params(DIMS, "relu", O.ORng(0))
    X, y = O.synthetic_batch(B, DIMS[0], DIMS[-1])
    bl = B // world
    Xs, ys = X[rank * bl:(rank + 1) * bl], y[rank * bl:(rank + 1) * bl]
    lin = O.linearize(DIMS, "relu", "ce", w, Xs, ys)
    scale = bl / B  # local means -> contributions to the global mean
    v = O.ORng(2).normal(w.size)
    parts = {
        "loss": np.array([lin.value * scale]),
        "grad": lin.grad * scale,
        "ggn": O.ggn_matvec(lin, v) * scale,
        "hvp": O.hvp(lin, v) * scale,
    }
    res = {}
    for k, a in parts.items():
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t)
        res[k] = t.numpy()
    # a replicated CG on the all-reduced operator takes identical decisions on every rank
    def mv(x):
        t = torch.from_numpy(O.ggn_matvec(lin, x) * scale)
        dist.all_reduce(t)
        return t.numpy()

    cg = O.cg(mv, res["grad"], 1.0, 1e-5, 10, 10)
    res["cg_x"] = cg.x
    res["cg_iters"] = np.array([cg.iterations])
    out[rank] = res
    dist.destroy_process_group()


def test_two_rank_sharding_matches_full_batch():
    from oracle import curvopt_oracle as O

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    w = O.init_params(DIMS, "relu", O.ORng(0))
    X, y = O.synthetic_batch(B, DIMS[0], DIMS[-1])
    lin = O.linearize(DIMS, "relu", "ce", w, X, y)
    v = O.ORng(2).normal(w.size)
    full = {"loss": np.array([lin.value]), "grad": lin.grad, "ggn": O.ggn_matvec(lin, v), "hvp": O.hvp(lin, v)}
    cg = O.cg(lambda x: O.ggn_matvec(lin, x), lin.grad, 1.0, 1e-5, 10, 10)
    for r in range(world):
        for k, ref in full.items():
            np.testing.assert_allclose(out[r][k], ref, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(out[r]["cg_x"], cg.x, rtol=1e-8, atol=1e-12)
        assert int(out[r]["cg_iters"][0]) == cg.iterations
    np.testing.assert_array_equal(out[0]["cg_x"], out[1]["cg_x"])


def test_bench_shards_cover_the_global_batch():
    sys.path.insert(0, ROOT)
    import bench

    full = bench.make_batches(1, 64, 0, 1)[0]
    shards = [bench.make_batches(1, 64, r, 4)[0] for r in range(4)]
    np.testing.assert_array_equal(np.concatenate([s[0] for s in shards]), full[0])
    np.testing.assert_array_equal(np.concatenate([s[1] for s in shards]), full[1])
