"""World-size-2 CPU tests (gloo) of the data-parallel step's host logic:

  (a) identical subgraphs on every rank: mean(dW) == single-rank dW,
  (b) different seeded subgraphs: mean over ranks of the oracle dW equals the mean of the
      per-rank fp64 dW computed on one rank,
  (c) world size 1 is the identity,
  plus the seed scheme (distinct subgraphs / inputs per rank, replicated weights) and the
  timing reduction (max over ranks, work summed).
The GPU path's gsg_allreduce_grads is the NCCL counterpart of the same mean (tested at N = 1
on the GPU box; only one GPU is available there).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as orc
        import workload as wl
        from paper_2010_03166_b200 import dp

        cfg = wl.tiny_config(n_parent=2000, mean_deg=8.0, n=96, m=24, dims=(8, 6), head="softmax", classes=5)
        res = {}
        # (b) different subgraphs per rank
        g = wl.sample_subgraph(cfg, 0, rank)
        inp = wl.make_inputs(cfg, g.n, 0, rank)
        A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
        out = orc.model_step(A, inp.X, inp.Ws, inp.W_mlp, inp.labels, "softmax")
        mean = dp.mean_grads_reference([out["dW"][0], out["dW_mlp"]])
        res["mean"] = [m.numpy() for m in mean]
        res["W0"] = inp.Ws[0]
        res["nodes"] = g.nodes
        # (a) identical subgraph on every rank
        g0 = wl.sample_subgraph(cfg, 0, 0)
        inp0 = wl.make_inputs(cfg, g0.n, 0, 0)
        A0 = orc.normalize(g0.indptr, g0.indices, orc.NORM_ROW_SELF)
        o0 = orc.model_step(A0, inp0.X, inp0.Ws, inp0.W_mlp, inp0.labels, "softmax")
        res["same_mean"] = dp.mean_grads_reference([o0["dW"][0]])[0].numpy()
        res["same_single"] = o0["dW"][0]
        # timing reduction
        res["timing"] = dp.reduce_timing(10.0 + rank, 100.0 * (rank + 1))
        uid = dp.broadcast_bytes(b"x" * 128 if rank == 0 else None)
        res["uid"] = uid
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_different_subgraphs_mean(results):
    import oracle as orc
    import workload as wl
    cfg = wl.tiny_config(n_parent=2000, mean_deg=8.0, n=96, m=24, dims=(8, 6), head="softmax", classes=5)
    per_rank = []
    for r in range(2):
        g = wl.sample_subgraph(cfg, 0, r)
        inp = wl.make_inputs(cfg, g.n, 0, r)
        A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
        o = orc.model_step(A, inp.X, inp.Ws, inp.W_mlp, inp.labels, "softmax")
        per_rank.append([o["dW"][0], o["dW_mlp"]])
    expect = [(per_rank[0][i] + per_rank[1][i]) / 2 for i in range(2)]
    for r in range(2):
        for got, exp in zip(results[r]["mean"], expect):
            np.testing.assert_allclose(got, exp, rtol=1e-12, atol=1e-12)


def test_identical_subgraphs_mean_is_single(results):
    for r in range(2):
        np.testing.assert_allclose(results[r]["same_mean"], results[r]["same_single"], rtol=1e-15, atol=1e-15)


def test_seed_scheme(results):
    assert not np.array_equal(results[0]["nodes"], results[1]["nodes"])  # own subgraph per rank
    np.testing.assert_array_equal(results[0]["W0"], results[1]["W0"])    # replicated weights


def test_timing_reduction(results):
    for r in range(2):
        assert results[r]["timing"] == (11.0, 300.0)  # max over ranks, work summed
        assert results[r]["uid"] == b"x" * 128


def test_world_size_one_is_identity():
    from paper_2010_03166_b200 import dp
    g = np.arange(6.0).reshape(2, 3)
    np.testing.assert_array_equal(dp.mean_grads_reference([g])[0].numpy(), g)
    assert dp.reduce_timing(3.0, 7.0) == (3.0, 7.0)
