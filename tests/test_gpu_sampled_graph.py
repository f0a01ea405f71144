"""GPU-sampled training under one CUDA graph (Alg. 7's pool refill, with Alg. 2 on the
device): gsg_sample_load copies sample *d_k of a gsg_frontier_sample batch
into a device-sized subgraph (every size on the device, padding nodes isolated), so a single
captured step -- load, X_s = X[V_s] gather, normalize, layers, head, backward -- serves every
sample of the batch.

  * the loaded subgraph equals the sample (structure of the real nodes = the oracle's induced
    subgraph of the sampler's node set, padding rows = their self loop only), nodes / loss
    weights as documented in gsg.h;
  * each graph replay trains on the next sample and gives the same loss and gradients as an
    eager step on that sample uploaded from the host without padding (1e-5);
  * a sample that does not fit is reported by gsg_sample_check.
"""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2010_03166_b200 as gsg
import workload as wl
from paper_2010_03166_b200.step import GCNStep

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    assert np.all(np.isfinite(a))
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def setup():
    cfg = wl.tiny_config(n_parent=6000, mean_deg=12.0, n=400, m=40, dims=(48, 64, 32), head="sigmoid", classes=12)
    p = wl.parent_for(cfg).csr()
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    batch = pg.sample(cfg.n, cfg.m, 777, count=3, clip=16)
    yield cfg, p, ctx, stream, pg, batch
    batch.free()
    pg.free()
    ctx.close()


def test_sample_load_structure(setup):
    cfg, p, ctx, stream, pg, batch = setup
    n_pad = 448
    sg = ctx.create_device(n_pad, 40000)
    d_k = torch.zeros(1, dtype=torch.int32, device="cuda")
    nodes = torch.full((n_pad,), 7, dtype=torch.int32, device="cuda")
    w = torch.full((n_pad,), 3.0, device="cuda")
    for k in range(4):  # wraps around: 0, 1, 2, 0
        with torch.cuda.stream(stream):
            batch.load(ctx, d_k, sg, nodes, w)
            sg.normalize()
        stream.synchronize()
        ip, ix, nd = batch.to_host(k % 3)
        nk = nd.size
        dip, dix, dval, _ = sg.download()
        ref = orc.normalize(ip, ix, orc.NORM_ROW_SELF)
        assert np.array_equal(dip[:nk + 1], ref.indptr) and np.array_equal(dix[:ref.idx.size], ref.idx)
        np.testing.assert_allclose(dval[:ref.val.size], ref.val, rtol=2 ** -23, atol=0)
        # padding nodes nk .. n_pad-1: the self loop only, weight 1
        assert np.array_equal(np.diff(dip[nk:]), np.ones(n_pad - nk))
        assert np.array_equal(dix[ref.idx.size:], np.arange(nk, n_pad))
        assert np.all(dval[ref.idx.size:] == 1.0)
        assert np.array_equal(nodes.cpu().numpy()[:nk], nd) and np.all(nodes.cpu().numpy()[nk:] == -1)
        wv = w.cpu().numpy()
        assert np.all(wv[:nk] == np.float32(1.0 / nk)) and np.all(wv[nk:] == 0)
        assert int(d_k.item()) == (k + 1) % 3
    batch.check()
    sg.free()


def test_graph_replay_trains_each_sample(setup):
    cfg, p, ctx, stream, pg, batch = setup
    n_pad = 416
    f0 = cfg.dims[0]
    rng = np.random.default_rng(3)
    Xpar = rng.standard_normal((p.n, f0)).astype(np.float32)
    Lpar = (rng.random((p.n, cfg.classes)) < 0.1).astype(np.uint8)
    inp = wl.make_inputs(cfg, 8)
    with torch.cuda.stream(stream):
        Xp = torch.zeros((p.n, wl.ld_for(f0)), device="cuda")[:, :f0]
        Xp.copy_(torch.from_numpy(Xpar))
        Lp = torch.from_numpy(Lpar).cuda()
        sg = ctx.create_device(n_pad, 40000)
        d_k = torch.zeros(1, dtype=torch.int32, device="cuda")
        nodes = torch.zeros((n_pad,), dtype=torch.int32, device="cuda")
        node_w = torch.zeros((n_pad,), device="cuda")
        Xs = torch.zeros((n_pad, wl.ld_for(f0)), device="cuda")[:, :f0]
        Ls = torch.zeros((n_pad, cfg.classes), dtype=torch.uint8, device="cuda")
        step = GCNStep(ctx, cfg.dims, n_pad, cfg.head, cfg.classes, cfg.precision, weights=inp.Ws, w_mlp=inp.W_mlp)

        def one():
            batch.load(ctx, d_k, sg, nodes, node_w)
            ctx.gather_rows(Xp, _ptr(nodes), Xs, n_pad)
            ctx.gather_rows(Lp, _ptr(nodes), Ls, n_pad)
            step.forward_backward(sg, Xs, labels=Ls, node_w=node_w)
        one()  # eager warm-up (workspaces), sample 0
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        one()
    ref_ctx = gsg.Context(0)
    for r in range(4):  # replays train samples 1, 2, 0, 1
        with torch.cuda.stream(stream):
            g.replay()
        stream.synchronize()
        k = (r + 1) % 3
        ip, ix, nd = batch.to_host(k)
        nk = nd.size
        # eager reference: the same sample uploaded from the host, n_k nodes, no padding, no weights
        rsg = ref_ctx.upload(ip, ix)
        rstep = GCNStep(ref_ctx, cfg.dims, nk, cfg.head, cfg.classes, cfg.precision, weights=inp.Ws, w_mlp=inp.W_mlp)
        X = torch.zeros((nk, wl.ld_for(f0)), device="cuda")[:, :f0]
        X.copy_(torch.from_numpy(Xpar[nd]))
        rstep.forward_backward(rsg, X, labels=torch.from_numpy(Lpar[nd]).cuda())
        ref_ctx.sync()
        assert abs(float(step.loss.item()) - float(rstep.loss.item())) <= 1e-5 * abs(float(rstep.loss.item()))
        for a, b in zip(step.dW + [step.dWm], rstep.dW + [rstep.dWm]):
            assert rel(a.cpu().numpy(), b.cpu().numpy()) <= 1e-5
        assert rel(step.H[-1][:nk].cpu().numpy(), rstep.H[-1][:nk].cpu().numpy()) <= 1e-5
        assert not step.H[-1][nk:].any()  # padding rows stay zero
        rsg.free()
    batch.check()
    sg.free()
    ref_ctx.close()


def test_sample_load_overflow_is_reported(setup):
    cfg, p, ctx, stream, pg, batch = setup
    sg = ctx.create_device(448, 10)  # far too few entries
    d_k = torch.zeros(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(stream):
        batch.load(ctx, d_k, sg)
    stream.synchronize()
    with pytest.raises(gsg.GsgError):
        batch.check()
    sg.free()


def _ptr(t):
    return t.data_ptr()


@pytest.mark.parametrize("dtype,cols,pitch", [(torch.float32, 200, 200), (torch.float32, 50, 56), (torch.uint8, 107, 107),
                                              (torch.uint8, 1, 3), (torch.uint8, 33, 48), (torch.int32, 1, 1)])
@pytest.mark.parametrize("rows", [1, 5, 1000])
def test_gather_rows_exact(dtype, cols, pitch, rows):
    """gsg_gather_rows == numpy fancy indexing, byte for byte (the 16-byte and the byte path, a
    partial last group of rows, padding rows idx = -1 written as zeros, destination padding
    columns untouched)."""
    rng = np.random.default_rng(rows * 31 + cols)
    n_src = 3000
    if dtype == torch.uint8:
        src_h = rng.integers(0, 256, (n_src, pitch), dtype=np.uint8)
    elif dtype == torch.int32:
        src_h = rng.integers(-2**31, 2**31 - 1, (n_src, pitch), dtype=np.int32)
    else:
        src_h = rng.standard_normal((n_src, pitch)).astype(np.float32)
    idx_h = rng.integers(0, n_src, rows).astype(np.int32)
    idx_h[rng.random(rows) < 0.1] = -1
    src = torch.from_numpy(src_h).cuda()[:, :cols]
    dst_full = torch.from_numpy(np.full((rows, pitch), 77, dtype=src_h.dtype)).cuda()
    dst = dst_full[:, :cols]
    idx = torch.from_numpy(idx_h).cuda()
    ctx = gsg.Context(0)
    ctx.gather_rows(src, idx.data_ptr(), dst, rows)
    ctx.sync()
    ref = np.where(idx_h[:, None] >= 0, src_h[np.maximum(idx_h, 0), :cols], 0).astype(src_h.dtype)
    got = dst_full.cpu().numpy()
    assert np.array_equal(got[:, :cols], ref)
    assert np.all(got[:, cols:] == 77)
    ctx.close()
