"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star; SURVEY §8(c) "GPU vs oracle"):
  * fp32 SpMM outputs (P = Â X, dX = Âᵀ T):      max|gpu - orc| / max|orc| <= 1e-5
  * TF32 / BF16 tensor-core GEMM outputs:        max|gpu - orc| / max|orc| <= 5e-3
  * integer / index work (Â structure, bins):    bit-exact; valT = Alg. 4 permutation of val, bit-exact
Stage-isolated: each GPU stage is compared with the oracle's stage fed the GPU's own inputs.
"""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2010_03166_b200 as gsg
import workload as wl

pytestmark = pytest.mark.gpu

SPMM_TOL = 1e-5
GEMM_TOL = 5e-3


def rel_err(gpu, ref):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (gpu.shape, ref.shape)
    assert np.all(np.isfinite(gpu)), "non-finite GPU output"
    den = np.abs(ref).max()
    return float(np.abs(gpu - ref).max() / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def ctx():
    c = gsg.Context(0)
    yield c
    c.close()


def dev(a: np.ndarray, ld: int | None = None, pad_nan: bool = True):
    """Row-major device copy with row stride ld (padding filled with NaN to catch leaks)."""
    a = np.ascontiguousarray(a, np.float32)
    r, f = a.shape
    ld = wl.ld_for(f) if ld is None else ld
    t = torch.full((r, ld), float("nan") if pad_nan else 0.0, dtype=torch.float32, device="cuda")
    t[:, :f] = torch.from_numpy(a).cuda()
    return t[:, :f]


def empty(r, f, ld=None):
    ld = wl.ld_for(f) if ld is None else ld
    return torch.full((r, ld), float("nan"), dtype=torch.float32, device="cuda")[:, :f]


def host(t):
    torch.cuda.synchronize()
    return t.float().cpu().numpy().astype(np.float64)


def graph(n_parent, deg, n, m, seed):
    p = wl.Parent(n_parent, deg, 2.1, 0.0, seed=seed)
    return p.frontier_sample(n, m, seed + 1, clip=1)


def star_plus_random(n, hub_deg, seed):
    """A graph with one hub of degree hub_deg (heavy row path) plus random sparse edges."""
    rng = np.random.default_rng(seed)
    E = set()
    for j in rng.choice(np.arange(1, n), size=hub_deg, replace=False):
        E.add((0, int(j))); E.add((int(j), 0))
    for _ in range(3 * n):
        a, b = rng.integers(1, n, 2)
        if a != b:
            E.add((int(a), int(b))); E.add((int(b), int(a)))
    E = sorted(E)
    ip = np.zeros(n + 1, np.int64)
    for a, _ in E:
        ip[a + 1] += 1
    ip = np.cumsum(ip)
    ix = np.array([b for _, b in E], np.int32)
    return wl.CSR(ip, ix)


# ------------------------------------------------------------------------------ a1
@pytest.mark.parametrize("mode", [gsg.GSG_NORM_ROW_SELF, gsg.GSG_NORM_SYM_SELF, gsg.GSG_NORM_ROW, gsg.GSG_NORM_VALUES])
def test_normalize_matches_oracle(ctx, mode):
    g = graph(3000, 10.0, 700, 60, 1)
    vals = wl.random_values(g, 5) if mode == gsg.GSG_NORM_VALUES else None
    sg = ctx.upload(g.indptr, g.indices, vals).normalize(mode)
    ip, ix, v, vt = sg.download()
    A = orc.normalize(g.indptr, g.indices, mode, vals)
    assert np.array_equal(ip, A.indptr) and np.array_equal(ix, A.idx)  # structure: bit-exact
    np.testing.assert_allclose(v, A.val, rtol=2 ** -23, atol=0)           # one fp32 rounding
    # valT must be exactly Alg. 4's DataTrans of the GPU's own values (a permutation)
    ref_t = orc.transpose_alg4(orc.AHat(ip, ix, v.astype(np.float64)))
    assert np.array_equal(vt.astype(np.float64), ref_t)
    inf = sg.info()
    d = np.diff(ip)
    assert inf["nnz_hat"] == A.val.size and inf["max_deg_hat"] == d.max()
    assert inf["n_heavy"] == int((d >= 256).sum())


def test_upload_validation(ctx):
    ok = wl.CSR(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32))
    ctx.upload(ok.indptr, ok.indices).free()
    bad = [
        (np.array([0, 1, 1], np.int64), np.array([1], np.int32), "not symmetric"),
        (np.array([0, 1, 2], np.int64), np.array([0, 1], np.int32), "self loop"),
        (np.array([0, 1, 2], np.int64), np.array([5, 0], np.int32), "out of range"),
        (np.array([0, 2, 4, 6], np.int64), np.array([2, 1, 0, 2, 0, 1], np.int32), "ascending"),
    ]
    for ip, ix, msg in bad:
        with pytest.raises(gsg.GsgError) as e:
            ctx.upload(ip, ix)
        assert e.value.code == gsg.GSG_EGRAPH and msg in str(e.value), str(e.value)


# ------------------------------------------------------------------------------ a2 / a7
@pytest.mark.parametrize("f", [1, 3, 13, 50, 64, 128, 200, 300, 602])
def test_spmm_forward_and_transpose(ctx, f):
    g = graph(4000, 12.0, 900, 80, 2)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_ROW_SELF)
    rng = np.random.default_rng(f)
    X = rng.standard_normal((g.n, f)).astype(np.float32)
    Xd, Y = dev(X), empty(g.n, f)
    ctx.spmm(sg, Xd, Y)
    assert rel_err(host(Y), orc.spmm(A, X)) <= SPMM_TOL
    Yt = empty(g.n, f)
    ctx.spmm(sg, Xd, Yt, transpose=True)
    assert rel_err(host(Yt), orc.spmm_t(A, X)) <= SPMM_TOL


@pytest.mark.parametrize("n,hub", [(3000, 2500), (12000, 9000)])
def test_spmm_heavy_rows_and_mask(ctx, n, hub):
    # hub degree >= 2048: a "mega" row, split over 8 CTAs per column chunk and combined in order
    g = star_plus_random(n, hub, 3)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_SYM_SELF)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_SYM_SELF)
    assert sg.info()["n_heavy"] >= 1
    rng = np.random.default_rng(4)
    for f in (8, 200, 1024):
        X = rng.standard_normal((g.n, f)).astype(np.float32)
        Hb = rng.standard_normal((g.n, f)).astype(np.float32)
        Y, Ylp = empty(g.n, f), torch.zeros((g.n, wl.ld_for(f, 8)), dtype=torch.bfloat16, device="cuda")[:, :f]
        ctx.spmm(sg, dev(X), Y, transpose=True, mask=dev(Hb), Ylp=Ylp)
        ref = np.where(Hb > 0, orc.spmm_t(A, X), 0.0)
        assert rel_err(host(Y), ref) <= SPMM_TOL
        yl = host(Ylp)
        assert np.array_equal(yl, torch.from_numpy(host(Y).astype(np.float32)).bfloat16().float().numpy())
        Y2 = empty(g.n, f)
        ctx.spmm(sg, dev(X), Y2, transpose=True, mask=dev(Hb))
        assert torch.equal(Y, Y2)  # the segment combine is order-fixed


@pytest.mark.parametrize("f", [65, 200, 300, 1024, 1100])
def test_spmm_dense_frontier(ctx, f):
    """Dense frontier subgraph (config-5-like density, heavy rows, many shared high-degree
    neighbors) at widths with full and ragged column chunks (f = 1100: 5 chunks of 55 float4)."""
    g = graph(20000, 40.0, 2500, 300, 11)
    d = np.diff(g.indptr) + 1
    assert (d >= 16).sum() > 300 and d.max() >= 256
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_ROW_SELF)
    rng = np.random.default_rng(100 + f)
    X = rng.standard_normal((g.n, f)).astype(np.float32)
    Y, Yt = empty(g.n, f), empty(g.n, f)
    ctx.spmm(sg, dev(X), Y)
    ctx.spmm(sg, dev(X), Yt, transpose=True)
    assert rel_err(host(Y), orc.spmm(A, X)) <= SPMM_TOL
    assert rel_err(host(Yt), orc.spmm_t(A, X)) <= SPMM_TOL
    Y2 = empty(g.n, f)
    ctx.spmm(sg, dev(X), Y2)
    assert torch.equal(Y, Y2)


@pytest.mark.gpu
@pytest.mark.parametrize("f", [260, 300, 320, 324, 384, 602, 1100])
def test_spmm_lane_group_tail(ctx, f):
    """The last column chunk gathered by lane groups (f4 mod 64 in [1, 32], 32-byte rows): group
    sizes 8 (r <= 16 float4: f = 260, 300, 320) and 16 (f = 324, 384, 602, 1100), at the group-size
    boundaries r = 1 / 16 / 17 / 32, on light rows, a CTA-split heavy row (degree 1,200 < the
    mega-row bound, f >= 1024 launches) and as warp segments, with the bitmask gate and the bf16
    copy, element-wise at 1e-5 and bitwise reproducible."""
    rng = np.random.default_rng(300 + f)
    for g, mode, orc_mode in ((graph(4000, 12.0, 900, 80, 2), gsg.GSG_NORM_ROW_SELF, orc.NORM_ROW_SELF),
                              (star_plus_random(6000, 1200, 8), gsg.GSG_NORM_SYM_SELF, orc.NORM_SYM_SELF)):
        A = orc.normalize(g.indptr, g.indices, orc_mode)
        sg = ctx.upload(g.indptr, g.indices).normalize(mode)
        X = rng.standard_normal((g.n, f)).astype(np.float32)
        Hb = rng.standard_normal((g.n, f)).astype(np.float32)
        Xd = dev(X)
        assert Xd.stride(0) % 8 == 0 and Xd.data_ptr() % 32 == 0  # the 256-bit gather path
        Y, Yt = empty(g.n, f), empty(g.n, f)
        Ylp = torch.zeros((g.n, wl.ld_for(f, 8)), dtype=torch.bfloat16, device="cuda")[:, :f]
        ctx.spmm(sg, Xd, Y)
        ctx.spmm(sg, Xd, Yt, transpose=True, mask=dev(Hb), Ylp=Ylp)
        assert rel_err(host(Y), orc.spmm(A, X)) <= SPMM_TOL
        ref_t = np.where(Hb > 0, orc.spmm_t(A, X), 0.0)
        assert rel_err(host(Yt), ref_t) <= SPMM_TOL
        assert np.array_equal(host(Ylp), torch.from_numpy(host(Yt).astype(np.float32)).bfloat16().float().numpy())
        Y2 = empty(g.n, f)
        ctx.spmm(sg, Xd, Y2)
        assert torch.equal(Y, Y2)


def test_spmm_deterministic_and_identity(ctx):
    g = graph(5000, 20.0, 1500, 100, 5)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    X = dev(np.random.default_rng(6).standard_normal((g.n, 256)).astype(np.float32))
    Y1, Y2 = empty(g.n, 256), empty(g.n, 256)
    ctx.spmm(sg, X, Y1)
    ctx.spmm(sg, X, Y2)
    assert torch.equal(Y1, Y2)
    # no edges: Â = I -> P = X exactly
    n = 37
    e = ctx.upload(np.zeros(n + 1, np.int64), np.zeros(0, np.int32)).normalize()
    Xi = np.random.default_rng(7).standard_normal((n, 20)).astype(np.float32)
    Yi = empty(n, 20)
    ctx.spmm(e, dev(Xi), Yi)
    assert np.array_equal(host(Yi), Xi.astype(np.float64))


def test_spmm_edge_cases(ctx):
    """Degenerate and boundary inputs: a subgraph with no nodes, a single node, argument errors
    (stride / alignment / aliasing) and the 32-bit byte-offset limit (n * ldx * 4 >= 4 GiB is
    refused with GSG_EUNSUPPORTED before anything is read)."""
    z = ctx.upload(np.zeros(1, np.int64), np.zeros(0, np.int32)).normalize()
    X0 = torch.zeros((0, 64), device="cuda")
    ctx.spmm(z, X0, torch.zeros((0, 64), device="cuda"))                    # n = 0: no-op
    one = ctx.upload(np.zeros(2, np.int64), np.zeros(0, np.int32)).normalize()
    X1 = dev(np.full((1, 300), 3.0, np.float32))
    Y1 = empty(1, 300)
    ctx.spmm(one, X1, Y1)
    assert np.array_equal(host(Y1), np.full((1, 300), 3.0))               # Â = [1]
    g = graph(3000, 10.0, 500, 60, 13)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    X = dev(np.ones((g.n, 64), np.float32))
    with pytest.raises(gsg.GsgError) as e:                                  # aliasing
        ctx.spmm(sg, X, X)
    assert e.value.code == gsg.GSG_EINVAL
    buf = torch.zeros(64 * g.n + 8, device="cuda")
    with pytest.raises(gsg.GsgError) as e:                                  # 16-byte alignment
        gsg.check(gsg.gsg_spmm(ctx.h, sg.h, 0, 64, buf.data_ptr() + 4, 64, empty(g.n, 64).data_ptr(), 64,
                               None, 0, None, 0, None, 0))
    assert e.value.code == gsg.GSG_EINVAL
    with pytest.raises(gsg.GsgError) as e:                                  # ld < f
        gsg.check(gsg.gsg_spmm(ctx.h, sg.h, 0, 64, buf.data_ptr(), 60, empty(g.n, 64).data_ptr(), 64,
                               None, 0, None, 0, None, 0))
    assert e.value.code == gsg.GSG_EINVAL
    big = ctx.upload(np.zeros((1 << 20) + 1, np.int64), np.zeros(0, np.int32)).normalize()
    with pytest.raises(gsg.GsgError) as e:                                  # 2^20 rows x 1024 x 4 B = 4 GiB
        gsg.check(gsg.gsg_spmm(ctx.h, big.h, 0, 1024, buf.data_ptr(), 1024, buf.data_ptr() + 4096, 1024,
                               None, 0, None, 0, None, 0))
    assert e.value.code == gsg.GSG_EUNSUPPORTED


# ------------------------------------------------------------------------------ GEMMs
GEMM_SHAPES = [(128, 128, 32), (300, 200, 50), (1000, 512, 602), (130, 17, 5), (602, 512, 3000), (64, 1024, 1024),
               (2000, 107, 1024)]


@pytest.mark.parametrize("prec", [gsg.GSG_PREC_TF32, gsg.GSG_PREC_BF16])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_vs_oracle(ctx, prec, ta, tb, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = orc.gemm(A, B, ta, tb)
    if prec == gsg.GSG_PREC_BF16:
        Ad = torch.from_numpy(A).cuda().bfloat16()
        Bd = torch.from_numpy(B).cuda().bfloat16()
        pa = torch.zeros((A.shape[0], wl.ld_for(A.shape[1], 8)), dtype=torch.bfloat16, device="cuda")
        pb = torch.zeros((B.shape[0], wl.ld_for(B.shape[1], 8)), dtype=torch.bfloat16, device="cuda")
        pa[:, :A.shape[1]] = Ad
        pb[:, :B.shape[1]] = Bd
        Ad, Bd = pa[:, :A.shape[1]], pb[:, :B.shape[1]]
    else:
        Ad, Bd = dev(A), dev(B)
    C = empty(M, N)
    ctx.gemm(Ad, Bd, C, transA=ta, transB=tb, precision=prec, K=K)
    assert rel_err(host(C), ref) <= GEMM_TOL


@pytest.mark.parametrize("split,ta", [(16, True), (40, True), (64, False)])
def test_gemm_splitk_many(ctx, split, ta):
    """Many K pieces and few outputs (head-gradient shapes, dW_mlp = H_L^T dS over K = n): the
    warp-per-output reduction, with the gate and bf16-copy epilogues, deterministic."""
    rng = np.random.default_rng(split)
    M, N, K = 512, 41, 8000
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    aux = rng.standard_normal((M, N)).astype(np.float32)
    ref = orc.gemm(A, B, ta, False)
    C, C2 = empty(M, N), empty(M, N)
    Clp = torch.zeros((M, wl.ld_for(N, 8)), dtype=torch.bfloat16, device="cuda")[:, :N]
    ctx.gemm(dev(A), dev(B), C, transA=ta, epilogue=gsg.GSG_EPI_MASK, aux=dev(aux), Clp=Clp, split_k=split, K=K)
    assert rel_err(host(C), np.where(aux > 0, ref, 0)) <= GEMM_TOL
    assert np.array_equal(host(Clp), torch.from_numpy(host(C).astype(np.float32)).bfloat16().float().numpy())
    ctx.gemm(dev(A), dev(B), C2, transA=ta, epilogue=gsg.GSG_EPI_MASK, aux=dev(aux), split_k=split, K=K)
    assert torch.equal(C, C2)


@pytest.mark.parametrize("split", [1, 3, 7])
def test_gemm_epilogues_and_splitk(ctx, split):
    rng = np.random.default_rng(11)
    M, N, K = 700, 300, 900
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    aux = rng.standard_normal((M, N)).astype(np.float32)
    ref = orc.gemm(A, B)
    C = empty(M, N)
    Clp = torch.zeros((M, wl.ld_for(N, 8)), dtype=torch.bfloat16, device="cuda")[:, :N]
    ctx.gemm(dev(A), dev(B), C, epilogue=gsg.GSG_EPI_RELU, Clp=Clp, split_k=split)
    assert rel_err(host(C), np.maximum(ref, 0)) <= GEMM_TOL
    assert np.array_equal(host(Clp), torch.from_numpy(host(C).astype(np.float32)).bfloat16().float().numpy())
    ctx.gemm(dev(A), dev(B), C, epilogue=gsg.GSG_EPI_MASK, aux=dev(aux), split_k=split)
    assert rel_err(host(C), np.where(aux > 0, ref, 0)) <= GEMM_TOL
    C0 = rng.standard_normal((M, N)).astype(np.float32)
    Cd = dev(C0)
    ctx.gemm(dev(A), dev(B), Cd, accumulate=True, split_k=split)
    assert rel_err(host(Cd), ref + C0) <= GEMM_TOL
    # bitwise reproducible
    C1, C2 = empty(M, N), empty(M, N)
    ctx.gemm(dev(A), dev(B), C1, split_k=split)
    ctx.gemm(dev(A), dev(B), C2, split_k=split)
    assert torch.equal(C1, C2)


def test_gemm_k0(ctx):
    C = dev(np.ones((5, 6), np.float32))
    A = empty(5, 4)
    ctx.gemm(A, A, C, K=0, M=5, N=6)
    assert not host(C).any()
    # M = 0 or N = 0: nothing to write, no pointer read (NULL accepted)
    for M, N in ((0, 16), (16, 0)):
        gsg.check(gsg.gsg_gemm(ctx.h, M, N, 32, None, 32, 0, None, 16, 0, None, 16, None, 0,
                               gsg.GSG_PREC_TF32, gsg.GSG_EPI_RELU, None, 0, None, 0, None, 0, 0, 0))


# ------------------------------------------------------------------------------ layer
def run_layer(ctx, g, X, W, dH, prec, mode=gsg.GSG_NORM_ROW_SELF, Hb=None):
    n, fi = X.shape
    fo = W.shape[1]
    sg = ctx.upload(g.indptr, g.indices).normalize(mode)
    Xd, Wd = dev(X), dev(W)
    P, H = empty(n, fi), empty(n, fo)
    Plp = torch.zeros((n, wl.ld_for(fi, 8)), dtype=torch.bfloat16, device="cuda")[:, :fi] if prec else None
    ctx.layer_forward(sg, Xd, Wd, P, H, fi, fo, precision=prec, Plp=Plp)
    dW, dX = empty(fi, fo), empty(n, fi)
    ctx.layer_backward(sg, P, H, dev(dH), Wd, dW, dX, fi, fo, precision=prec, Plp=Plp,
                       H_below=None if Hb is None else dev(Hb))
    return {k: host(v) for k, v in dict(P=P, H=H, dW=dW, dX=dX).items()}


@pytest.mark.parametrize("prec", [gsg.GSG_PREC_TF32, gsg.GSG_PREC_BF16])
def test_layer_stage_isolated(ctx, prec):
    cfg = wl.CONFIGS[1]
    g = wl.sample_subgraph(cfg)
    inp = wl.make_inputs(cfg, g.n)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    Hb = np.random.default_rng(3).standard_normal(inp.X.shape).astype(np.float32)
    out = run_layer(ctx, g, inp.X, inp.Ws[0], inp.dH, prec, Hb=Hb)
    assert rel_err(out["P"], orc.spmm(A, inp.X)) <= SPMM_TOL                       # a2
    assert rel_err(out["H"], np.maximum(orc.gemm(out["P"], inp.Ws[0]), 0)) <= GEMM_TOL   # a3 (GPU's P)
    dZ = orc.relu_mask(inp.dH, out["H"])                                            # a4 (GPU's H)
    assert rel_err(out["dW"], orc.gemm(out["P"], dZ, transA=True)) <= GEMM_TOL     # a5
    T = orc.gemm(dZ, inp.Ws[0], transB=True)                                        # a6 (oracle)
    assert rel_err(out["dX"], np.where(Hb > 0, orc.spmm_t(A, T), 0)) <= GEMM_TOL    # a7 after a TF32 GEMM


def test_layer_backward_concurrent_splitk(ctx):
    """Shapes where both backward GEMMs cut K (dW: 2 tiles, K = n; T: 8 tiles, K = 512) while
    dW runs on the side stream next to T -> dX: each stream has its own split-K workspace."""
    g = graph(4000, 12.0, 1000, 80, 31)
    fi, fo = 64, 512
    rng = np.random.default_rng(32)
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    W = (rng.standard_normal((fi, fo)) * 0.05).astype(np.float32)
    dH = rng.standard_normal((g.n, fo)).astype(np.float32)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    for _ in range(2):
        out = run_layer(ctx, g, X, W, dH, gsg.GSG_PREC_TF32)
        dZ = orc.relu_mask(dH, out["H"])
        assert rel_err(out["dW"], orc.gemm(out["P"], dZ, transA=True)) <= GEMM_TOL
        assert rel_err(out["dX"], orc.spmm_t(A, orc.gemm(dZ, W, transB=True))) <= GEMM_TOL


@pytest.mark.parametrize("order2", [False, True])
def test_layer_w_bf16_flag(ctx, order2):
    """GSG_W_BF16: a caller-owned bf16 copy of W (made once, shared by forward and backward) gives
    bit-identical results to the per-call conversion, in both chain orders."""
    g = graph(4000, 12.0, 900, 80, 21)
    fi, fo = (96, 64) if order2 else (64, 96)
    rng = np.random.default_rng(22)
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    W = (rng.standard_normal((fi, fo)) * 0.1).astype(np.float32)
    dH = rng.standard_normal((g.n, fo)).astype(np.float32)
    Hb = rng.standard_normal((g.n, fi)).astype(np.float32)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    Xd, Wd, dHd, Hbd = dev(X), dev(W), dev(dH), dev(Hb)
    Wl = torch.zeros((fi, wl.ld_for(fo, 8)), dtype=torch.bfloat16, device="cuda")[:, :fo]
    ctx.to_bf16(Wd, Wl)
    f2 = gsg.GSG_ORDER_A_XW if order2 else 0
    outs = []
    for Wop, fl in ((Wd, 0), (Wl, gsg.GSG_W_BF16)):
        P = empty(g.n, fo if order2 else fi)
        H = empty(g.n, fo)
        Plp = torch.zeros((g.n, wl.ld_for(fi, 8)), dtype=torch.bfloat16, device="cuda")[:, :fi]
        ctx.layer_forward(sg, Xd, Wop, P, H, fi, fo, precision=gsg.GSG_PREC_BF16, Plp=None if order2 else Plp,
                          flags=f2 | fl)
        if order2:
            ctx.to_bf16(Xd, Plp)
        dW, dX = empty(fi, fo), empty(g.n, fi)
        ctx.layer_backward(sg, Xd if order2 else P, H, dHd, Wop, dW, dX, fi, fo, precision=gsg.GSG_PREC_BF16,
                           Plp=Plp, H_below=Hbd, flags=f2 | fl)
        outs.append([host(t) for t in (H, dW, dX)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    with pytest.raises(gsg.GsgError) as e:      # bf16 W with a misaligned stride is refused
        bad = torch.zeros((fi, fo + 3), dtype=torch.bfloat16, device="cuda")[:, :fo]
        ctx.layer_forward(sg, Xd, bad, empty(g.n, fi), empty(g.n, fo), fi, fo, precision=gsg.GSG_PREC_BF16,
                          Plp=Plp, flags=gsg.GSG_W_BF16)
    assert e.value.code == gsg.GSG_EINVAL


@pytest.mark.parametrize("prec,order2", [(gsg.GSG_PREC_TF32, False), (gsg.GSG_PREC_BF16, False),
                                          (gsg.GSG_PREC_BF16, True), (gsg.GSG_PREC_FP32X3, False)])
def test_layer_h_bits_flag(ctx, prec, order2):
    """GSG_H_BITS: the backward's own dZ = dH ⊙ 1[H > 0] gate read from the forward's ReLU bitmask
    (d_H = H's bits) gives bit-identical dW and dX to the fp32-H gate, at a width with a partial
    last word (f_out = 100)."""
    g = graph(4000, 12.0, 900, 80, 23)
    fi, fo = (96, 100) if not order2 else (128, 100)
    rng = np.random.default_rng(24)
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    W = (rng.standard_normal((fi, fo)) * 0.1).astype(np.float32)
    dH = rng.standard_normal((g.n, fo)).astype(np.float32)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    Xd, Wd, dHd = dev(X), dev(W), dev(dH)
    bf = prec == gsg.GSG_PREC_BF16
    f2 = gsg.GSG_ORDER_A_XW if order2 else 0
    P = empty(g.n, fo if order2 else fi)
    H = empty(g.n, fo)
    Hbits = torch.zeros((g.n, (fo + 31) // 32), dtype=torch.int32, device="cuda")
    Plp = torch.zeros((g.n, wl.ld_for(fi, 8)), dtype=torch.bfloat16, device="cuda")[:, :fi] if bf else None
    ctx.layer_forward(sg, Xd, Wd, P, H, fi, fo, precision=prec, Plp=None if order2 else Plp, flags=f2,
                      H_bits=Hbits)
    if order2 and bf:
        ctx.to_bf16(Xd, Plp)
    outs = []
    for Hop, fl in ((H, 0), (Hbits, gsg.GSG_H_BITS)):
        dW, dX = empty(fi, fo), empty(g.n, fi)
        ctx.layer_backward(sg, Xd if order2 else P, Hop, dHd, Wd, dW, dX, fi, fo, precision=prec, Plp=Plp,
                           flags=f2 | fl)
        outs.append([host(t) for t in (dW, dX)])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
    Hh = host(H)
    dZ = np.where(Hh > 0, dH, 0.0)
    ref_dW = orc.gemm(orc.spmm(orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF), X), dZ, transA=True) \
        if not order2 else None
    if ref_dW is not None:
        assert rel_err(outs[1][0], ref_dW) <= GEMM_TOL


def test_layer_end_to_end_config1(ctx):
    cfg = wl.CONFIGS[1]
    g = wl.sample_subgraph(cfg)
    inp = wl.make_inputs(cfg, g.n)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    out = run_layer(ctx, g, inp.X, inp.Ws[0], inp.dH, gsg.GSG_PREC_TF32)
    P, Z, H = orc.layer_forward(A, inp.X, inp.Ws[0])
    assert rel_err(out["H"], H) <= GEMM_TOL
    # End to end (oracle from the initial inputs), the ReLU' gate may flip only where the TF32
    # pre-activation error can change the sign: |Z| within the GEMM tolerance of zero.
    flips = (out["H"] > 0) != (Z > 0)
    assert np.all(np.abs(Z[flips]) <= GEMM_TOL * np.abs(Z).max())
    assert flips.mean() < 1e-3
    # With the gate taken from the GPU's H (the only discontinuity), dW and dX agree at the
    # GEMM tolerance; each flipped gate moves dW by one P[k,i]*dH[k,j] term (not graded).
    dZ, dW, T, dX = orc.layer_backward(A, P, Z, np.where(out["H"] > 0, inp.dH, 0.0), inp.Ws[0], premasked=True)
    assert rel_err(out["dW"], dW) <= GEMM_TOL
    assert rel_err(out["dX"], dX) <= GEMM_TOL


@pytest.mark.parametrize("prec", [gsg.GSG_PREC_TF32, gsg.GSG_PREC_BF16])
def test_layer_chain_order2(ctx, prec):
    """§7.1 order 2, GSG_ORDER_A_XW: Y = X W, H = ReLU(Â Y); G = Âᵀ dZ, dW = Xᵀ G,
    dX = (G Wᵀ) ⊙ 1[H_below > 0] -- stage-isolated against the oracle's definitions."""
    g = graph(6000, 12.0, 1200, 100, 9)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    rng = np.random.default_rng(10)
    fi, fo = 300, 136
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    W = wl.glorot(rng, fi, fo)
    dH = rng.standard_normal((g.n, fo)).astype(np.float32)
    Hb = rng.standard_normal((g.n, fi)).astype(np.float32)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    Xd, Wd = dev(X), dev(W)
    Y, H = empty(g.n, fo), empty(g.n, fo)
    ctx.layer_forward(sg, Xd, Wd, Y, H, fi, fo, precision=prec, flags=gsg.GSG_ORDER_A_XW)
    Yg = host(Y)
    assert rel_err(Yg, orc.gemm(X, W)) <= GEMM_TOL
    Hg = host(H)
    assert rel_err(Hg, np.maximum(orc.spmm(A, Yg), 0)) <= SPMM_TOL
    Xlp = None
    if prec == gsg.GSG_PREC_BF16:
        Xlp = torch.zeros((g.n, wl.ld_for(fi, 8)), dtype=torch.bfloat16, device="cuda")[:, :fi]
        ctx.to_bf16(Xd, Xlp)
    dW, dX = empty(fi, fo), empty(g.n, fi)
    ctx.layer_backward(sg, Xd, H, dev(dH), Wd, dW, dX, fi, fo, precision=prec, Plp=Xlp, H_below=dev(Hb),
                       flags=gsg.GSG_ORDER_A_XW)
    dZ = orc.relu_mask(dH, Hg)
    assert rel_err(host(dW), orc.gemm(orc.spmm(A, X), dZ, transA=True)) <= GEMM_TOL
    assert rel_err(host(dX), np.where(Hb > 0, orc.spmm_t(A, orc.gemm(dZ, W, transB=True)), 0)) <= GEMM_TOL


@pytest.mark.parametrize("f", [8, 200, 512])
def test_spmm_weighted_adjacency(ctx, f):
    """General weighted Â (GSG_NORM_VALUES: GraphSAINT-style aggregator normalization):
    Âᵀ comes from the binary-search gather form of Alg. 4, not a closed form."""
    g = graph(5000, 14.0, 1100, 90, 12)
    vals = wl.random_values(g, 13)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_VALUES, vals)
    sg = ctx.upload(g.indptr, g.indices, vals).normalize(gsg.GSG_NORM_VALUES)
    X = np.random.default_rng(f).standard_normal((g.n, f)).astype(np.float32)
    Y, Yt = empty(g.n, f), empty(g.n, f)
    ctx.spmm(sg, dev(X), Y)
    ctx.spmm(sg, dev(X), Yt, transpose=True)
    assert rel_err(host(Y), orc.spmm(A, X)) <= SPMM_TOL
    assert rel_err(host(Yt), orc.spmm_t(A, X)) <= SPMM_TOL


@pytest.mark.parametrize("fi,fh", [(52, 16), (300, 128)])
def test_sage_layer(ctx, fi, fh):
    """GraphSAGE layer (NEXT #2; Eq. 1, Eqs. 12-15), stage-isolated."""
    g = graph(6000, 10.0, 1500, 120, 14)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW)
    rng = np.random.default_rng(fi)
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    Ws, Wn = wl.glorot(rng, fi, fh), wl.glorot(rng, fi, fh)
    dH = rng.standard_normal((g.n, 2 * fh)).astype(np.float32)
    Hb = rng.standard_normal((g.n, fi)).astype(np.float32)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_ROW)
    Xd, Wsd, Wnd = dev(X), dev(Ws), dev(Wn)
    P, H = empty(g.n, fi), empty(g.n, 2 * fh)
    ctx.sage_forward(sg, Xd, Wsd, Wnd, P, H, fi, fh)
    Pg, Hg = host(P), host(H)
    assert rel_err(Pg, orc.spmm(A, X)) <= SPMM_TOL
    assert rel_err(Hg, np.maximum(np.hstack([orc.gemm(X, Ws), orc.gemm(Pg, Wn)]), 0)) <= GEMM_TOL
    dWs, dWn, dX = empty(fi, fh), empty(fi, fh), empty(g.n, fi)
    ctx.sage_backward(sg, Xd, P, H, dev(dH), Wsd, Wnd, dWs, dWn, dX, fi, fh, H_below=dev(Hb))
    dZ = orc.relu_mask(dH, Hg)
    _, rWs, rWn, rX = orc.sage_backward(A, X, Pg, Hg, dZ, Ws, Wn, premasked=True)
    assert rel_err(host(dWs), rWs) <= GEMM_TOL
    assert rel_err(host(dWn), rWn) <= GEMM_TOL
    assert rel_err(host(dX), np.where(Hb > 0, rX, 0)) <= GEMM_TOL


@pytest.mark.parametrize("kind,C", [("softmax", 41), ("sigmoid", 107)])
def test_head_stage_isolated(ctx, kind, C):
    rng = np.random.default_rng(8)
    n, f = 1500, 200
    HL = np.maximum(rng.standard_normal((n, f)), 0).astype(np.float32)
    Wm = wl.glorot(rng, f, C) * 8
    labels = rng.integers(0, C, n).astype(np.int32) if kind == "softmax" else (rng.random((n, C)) < 0.05).astype(np.uint8)
    lab = torch.from_numpy(labels).cuda()
    S, dS = empty(n, C), empty(n, C)
    ldS = S.stride(0)
    dS = torch.full((n, ldS), float("nan"), device="cuda")[:, :C]
    dWm, dHL = empty(f, C), empty(n, f)
    loss = torch.zeros(1, device="cuda")
    HLd = dev(HL)
    ctx.head(HLd, dev(Wm), lab, S, dS, dWm, dHL, n, f, C,
             gsg.GSG_HEAD_SOFTMAX if kind == "softmax" else gsg.GSG_HEAD_SIGMOID, loss)
    Sg = host(S)
    assert rel_err(Sg, orc.gemm(HL, Wm)) <= GEMM_TOL
    l_ref, Y, dS_ref = orc.head(Sg, labels, kind)           # oracle fed the GPU's S
    assert abs(float(host(loss)[0]) - l_ref) <= 1e-5 * abs(l_ref)
    assert rel_err(host(dS), dS_ref) <= 1e-5
    dSg = host(dS)
    assert rel_err(host(dWm), orc.gemm(HL, dSg, transA=True)) <= GEMM_TOL
    assert rel_err(host(dHL), np.where(HL > 0, orc.gemm(dSg, Wm, transB=True), 0)) <= GEMM_TOL


def test_head_node_weights(ctx):
    """GraphSAINT-weighted loss (NEXT #4): loss = Σ λ_i CE_i, dS_i = λ_i (Y_i − Ȳ_i) ⊙ 1[S_i > 0]."""
    rng = np.random.default_rng(15)
    n, f, C = 900, 64, 20
    HL = np.maximum(rng.standard_normal((n, f)), 0).astype(np.float32)
    Wm = wl.glorot(rng, f, C) * 6
    labels = (rng.random((n, C)) < 0.1).astype(np.uint8)
    lam = rng.uniform(0.2, 2.0, n).astype(np.float32) / n
    S, dWm, dHL = empty(n, C), empty(f, C), empty(n, f)
    dS = torch.full((n, S.stride(0)), float("nan"), device="cuda")[:, :C]
    loss = torch.zeros(1, device="cuda")
    ctx.head(dev(HL), dev(Wm), torch.from_numpy(labels).cuda(), S, dS, dWm, dHL, n, f, C, gsg.GSG_HEAD_SIGMOID, loss,
             node_w=torch.from_numpy(lam).cuda())
    l_ref, _, dS_ref = orc.head(host(S), labels, "sigmoid", lam)
    assert abs(float(host(loss)[0]) - l_ref) <= 1e-5 * abs(l_ref)
    assert rel_err(host(dS), dS_ref) <= 1e-5


def test_allreduce_single_rank(ctx):
    uid = ctx.nccl_unique_id()
    comm = ctx.nccl_comm_init(1, 0, uid)
    a = torch.arange(1000, dtype=torch.float32, device="cuda")
    b = torch.ones(77, dtype=torch.float32, device="cuda")
    ref_a, ref_b = a.clone(), b.clone()
    ctx.allreduce_grads(comm, [a, b], average=True)
    ctx.sync()
    assert torch.equal(a, ref_a) and torch.equal(b, ref_b)
    ctx.nccl_comm_destroy(comm)


def test_spmm_largest_offsets(ctx):
    """Maximum size for the kernel's 32-bit row byte offsets: n * ldx * 4 just below 4 GiB
    (n = 1,048,575 rows of 1024 fp32). Isolated rows (Â_ii = 1) must come back exactly; a
    mega row (deg' = 2101 >= 2048: split over 8 CTAs per chunk) at the very end, whose neighbors
    span the whole address range, and its deg-1 neighbors are checked against fp64 sums."""
    f, n = 1024, (1 << 32) // (1024 * 4) - 1
    hub = n - 1
    nb = np.unique(np.linspace(0, n - 2, 2100).astype(np.int64))
    rows = np.concatenate([np.repeat(nb, 1), np.full(nb.size, hub)])
    cols = np.concatenate([np.full(nb.size, hub), nb])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    ip = np.zeros(n + 1, np.int64)
    np.add.at(ip, rows + 1, 1)
    ip = np.cumsum(ip)
    sg = ctx.upload(ip, cols.astype(np.int32)).normalize()
    X = torch.empty((n, f), device="cuda").normal_(generator=torch.Generator("cuda").manual_seed(5))
    Y = torch.empty((n, f), device="cuda")
    probe = np.array([1, 2, n // 3 + 1, n - 3], np.int64)       # isolated rows (not in nb)
    probe = probe[~np.isin(probe, nb)]
    for tr in (False, True):
        ctx.spmm(sg, X, Y, transpose=tr)
        torch.cuda.synchronize()
        pi = torch.from_numpy(probe).cuda()
        assert torch.equal(Y[pi], X[pi])
        nbt = torch.from_numpy(nb).cuda()
        Xn = X[nbt].double().cpu().numpy()
        Xh = X[hub].double().cpu().numpy()
        # row-self normalization: hub row 1/(deg+1) for itself and every neighbor (a2); the
        # transposed values (a7) take each entry's column degree: 1/2 for every neighbor
        ref_hub = (Xh + Xn.sum(0)) / (nb.size + 1) if not tr else Xh / (nb.size + 1) + Xn.sum(0) / 2
        got = Y[hub].double().cpu().numpy()
        assert np.abs(got - ref_hub).max() <= 1e-5 * np.abs(ref_hub).max()
        k = nb[-5:]
        ref_nb = (X[torch.from_numpy(k).cuda()].double().cpu().numpy() + Xh) / 2 if not tr else \
            X[torch.from_numpy(k).cuda()].double().cpu().numpy() / 2 + Xh / (nb.size + 1)
        got = Y[torch.from_numpy(k).cuda()].double().cpu().numpy()
        assert np.abs(got - ref_nb).max() <= 1e-5 * np.abs(ref_nb).max()
    del X, Y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("ta", [False, True])
def test_gemm_many_rows(ctx, ta):
    """A GEMM over a million-row operand (M = 1,048,575 x N = 96 x K = 40 and its transposed
    reduction form K = 1,048,575): 64-bit row offsets in every epilogue / split-K path; sampled
    rows / the full small output against fp64."""
    g = torch.Generator("cuda").manual_seed(9)
    big, small = (1 << 20) - 1, 40
    A = torch.empty((big, small), device="cuda").normal_(generator=g)
    B = torch.empty((big if ta else small, 96), device="cuda").normal_(generator=g)
    if not ta:
        C = torch.empty((big, 96), device="cuda")
        ctx.gemm(A, B, C, epilogue=gsg.GSG_EPI_RELU)
        idx = torch.tensor([0, 1, big // 2, big - 2, big - 1], device="cuda")
        ref = np.maximum(A[idx].double().cpu().numpy() @ B.double().cpu().numpy(), 0)
        assert rel_err(host(C[idx]), ref) <= GEMM_TOL
    else:
        C = torch.empty((small, 96), device="cuda")
        ctx.gemm(A, B, C, transA=True)                             # C = Aᵀ B, K = big (split-K)
        ref = A.double().T @ B.double()
        assert rel_err(host(C), ref.cpu().numpy()) <= GEMM_TOL


@pytest.mark.parametrize("f,ld,off", [(68, 68, 0), (300, 300, 0), (1100, 1100, 0), (1024, 1024, 4), (200, 204, 0)])
def test_spmm_128bit_gather_path(ctx, f, ld, off):
    """Operands the 256-bit gather path does not take (row stride not a multiple of 8 floats, or
    X only 16-byte aligned: `off` floats into the allocation) run the 128-bit wide path --
    light, heavy and mega rows (a 2500-degree hub), forward and transposed, with a mask."""
    g = star_plus_random(3000, 2500, 17)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_ROW_SELF)
    rng = np.random.default_rng(f + ld + off)
    X = rng.standard_normal((g.n, f)).astype(np.float32)
    Hb = rng.standard_normal((g.n, f)).astype(np.float32)
    buf = torch.full((g.n * ld + off,), float("nan"), device="cuda")
    Xd = buf[off:].view(g.n, ld)[:, :f]
    Xd.copy_(torch.from_numpy(X))
    Y = torch.full((g.n, ld), float("nan"), device="cuda")[:, :f]
    ctx.spmm(sg, Xd, Y)
    assert rel_err(host(Y), orc.spmm(A, X)) <= SPMM_TOL
    ctx.spmm(sg, Xd, Y, transpose=True, mask=dev(Hb))
    assert rel_err(host(Y), np.where(Hb > 0, orc.spmm_t(A, X), 0.0)) <= SPMM_TOL


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_gemm_strides_multiple_of_4(ctx, ta, tb):
    """TF32 operands and C with row strides that are multiples of 4 floats but not of 8 (TMA's
    16-byte rule is the only requirement), all three epilogues."""
    rng = np.random.default_rng(31)
    M, N, K = 700, 300, 420
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    aux = rng.standard_normal((M, N)).astype(np.float32)

    def dev4(a):
        r, c = a.shape
        ld = (c + 3) // 4 * 4 + (4 if ((c + 3) // 4 * 4) % 8 == 0 else 0)   # ld % 8 == 4
        return dev(a, ld)
    ref = orc.gemm(A, B, transA=ta, transB=tb)
    for epi, want in ((gsg.GSG_EPI_NONE, ref), (gsg.GSG_EPI_RELU, np.maximum(ref, 0)),
                      (gsg.GSG_EPI_MASK, np.where(aux > 0, ref, 0))):
        C = dev4(np.zeros((M, N), np.float32))
        assert C.stride(0) % 8 == 4
        ctx.gemm(dev4(A), dev4(B), C, transA=ta, transB=tb, epilogue=epi,
                 aux=dev4(aux) if epi == gsg.GSG_EPI_MASK else None, K=K)
        assert rel_err(host(C), want) <= GEMM_TOL
