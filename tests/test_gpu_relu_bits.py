"""ReLU bitmasks (include/gsg.h "ReLU bitmask"): the forward's ReLU epilogues write 1[H > 0] as one
bit per element and the backward's ReLU' gates (dZ = dH ⊙ σ'(Z)) read the bits instead of
the fp32 H. Pins: the written bits equal 1[H > 0] of the written H (bit-exact, packed here on the
host from the GPU's own H), and every gated result computed from the bits is bit-identical to the
same call gated by the fp32 matrix (which the other parity tests pin to the oracle).
"""
import numpy as np
import pytest
import torch

import paper_2010_03166_b200 as gsg
import workload as wl
from paper_2010_03166_b200.step import GCNStep

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = gsg.Context(0)
    yield c
    c.close()


def dev(a, ld=None):
    a = np.ascontiguousarray(a, np.float32)
    r, f = a.shape
    ld = wl.ld_for(f) if ld is None else ld
    t = torch.full((r, ld), float("nan"), dtype=torch.float32, device="cuda")
    t[:, :f] = torch.from_numpy(a).cuda()
    return t[:, :f]


def empty(r, f):
    return torch.full((r, wl.ld_for(f)), float("nan"), dtype=torch.float32, device="cuda")[:, :f]


def words(f):
    return (f + 31) // 32


def bits_buf(r, f, pad=1):
    """n x ceil(f/32) words inside an n x (ceil(f/32) + pad) buffer pre-filled with garbage (all
    ones) so a word the writer skips shows up; the pad words must stay untouched."""
    return torch.full((r, words(f) + pad), -1, dtype=torch.int32, device="cuda")[:, :words(f)]


def pack(H):
    """Host packing of 1[H > 0] in the gsg.h layout (bit i of word w = column 32 w + i)."""
    H = np.asarray(H)
    n, f = H.shape
    b = np.zeros((n, words(f) * 32), np.uint64)
    b[:, :f] = H > 0
    return (b.reshape(n, words(f), 32) << np.arange(32, dtype=np.uint64)).sum(-1).astype(np.uint32)


def hbits(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def h(t):
    torch.cuda.synchronize()
    return t.float().cpu().numpy()


def graph(n_parent, deg, n, m, seed):
    return wl.Parent(n_parent, deg, 2.1, 0.0, seed=seed).frontier_sample(n, m, seed + 1, clip=1)


@pytest.mark.parametrize("prec", [gsg.GSG_PREC_TF32, gsg.GSG_PREC_BF16])
@pytest.mark.parametrize("M,N,K", [(700, 300, 900), (500, 100, 64), (1000, 1024, 256), (333, 33, 40)])
def test_gemm_relu_bits_out(ctx, prec, M, N, K):
    rng = np.random.default_rng(M + N)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    Ad, Bd = dev(A), dev(B)
    if prec == gsg.GSG_PREC_BF16:
        Al = torch.zeros((M, wl.ld_for(K, 8)), dtype=torch.bfloat16, device="cuda")[:, :K]
        Bl = torch.zeros((K, wl.ld_for(N, 8)), dtype=torch.bfloat16, device="cuda")[:, :N]
        ctx.to_bf16(Ad, Al)
        ctx.to_bf16(Bd, Bl)
        Ad, Bd = Al, Bl
    C, Cb = empty(M, N), bits_buf(M, N)
    ctx.gemm(Ad, Bd, C, precision=prec, epilogue=gsg.GSG_EPI_RELU, C_bits=Cb, split_k=3)  # split forced to 1
    assert np.array_equal(hbits(Cb), pack(h(C)))
    full = torch.as_strided(Cb, (M, words(N) + 1), (Cb.stride(0), 1))
    assert np.all(hbits(full)[:, -1] == 0xFFFFFFFF)  # pad words untouched
    C2 = empty(M, N)
    ctx.gemm(Ad, Bd, C2, precision=prec, epilogue=gsg.GSG_EPI_RELU, split_k=1)
    assert torch.equal(C, C2)  # writing the bits does not change C


def test_gemm_relu_bits_k0(ctx):
    C, Cb = empty(40, 70), bits_buf(40, 70)
    ctx.gemm(dev(np.zeros((40, 8))), dev(np.zeros((8, 70))), C, epilogue=gsg.GSG_EPI_RELU, C_bits=Cb, K=0)
    assert np.all(hbits(Cb) == 0) and np.all(h(C) == 0)


@pytest.mark.parametrize("split", [1, 3, 7])
@pytest.mark.parametrize("prec,ta", [(gsg.GSG_PREC_TF32, False), (gsg.GSG_PREC_TF32, True), (gsg.GSG_PREC_BF16, False)])
@pytest.mark.parametrize("M,N,K", [(700, 300, 900), (2000, 1024, 107), (300, 45, 512)])
def test_gemm_mask_bits_equals_mask(ctx, split, prec, ta, M, N, K):
    rng = np.random.default_rng(7 * M + N)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    aux = rng.standard_normal((M, N)).astype(np.float32)
    aux[rng.random((M, N)) < 0.1] = 0.0   # exact zeros gate like negatives (1[aux > 0])
    Ad, Bd = dev(A), dev(B)
    if prec == gsg.GSG_PREC_BF16:
        Al = torch.zeros((M, wl.ld_for(K, 8)), dtype=torch.bfloat16, device="cuda")[:, :K]
        Bl = torch.zeros((K, wl.ld_for(N, 8)), dtype=torch.bfloat16, device="cuda")[:, :N]
        ctx.to_bf16(Ad, Al)
        ctx.to_bf16(Bd, Bl)
        Ad, Bd = Al, Bl
    ab = torch.from_numpy(pack(aux).view(np.int32)).cuda()
    C1, C2 = empty(M, N), empty(M, N)
    kw = dict(transA=ta, precision=prec, epilogue=gsg.GSG_EPI_MASK, split_k=split, K=K)
    ctx.gemm(Ad, Bd, C1, aux=dev(aux), **kw)
    ctx.gemm(Ad, Bd, C2, aux_bits=ab, **kw)
    assert torch.equal(C1, C2)


def star_plus_random(n, hub_deg, seed):
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
    return wl.CSR(np.cumsum(ip), np.array([b for _, b in E], np.int32))


@pytest.mark.parametrize("f", [8, 13, 64, 200, 1024, 1100])
def test_spmm_mask_bits_equals_mask(ctx, f):
    """All SpMM paths (narrow lane groups, wide chunks, heavy CTA-split and mega rows) gate from bits."""
    g = star_plus_random(3000, 2500, 5)
    sg = ctx.upload(g.indptr, g.indices).normalize(gsg.GSG_NORM_SYM_SELF)
    rng = np.random.default_rng(f)
    X = rng.standard_normal((g.n, f)).astype(np.float32)
    Hb = rng.standard_normal((g.n, f)).astype(np.float32)
    mb = torch.from_numpy(pack(Hb).view(np.int32)).cuda()
    Y1, Y2 = empty(g.n, f), empty(g.n, f)
    L1 = torch.zeros((g.n, wl.ld_for(f, 8)), dtype=torch.bfloat16, device="cuda")[:, :f]
    L2 = torch.zeros((g.n, wl.ld_for(f, 8)), dtype=torch.bfloat16, device="cuda")[:, :f]
    ctx.spmm(sg, dev(X), Y1, transpose=True, mask=dev(Hb), Ylp=L1)
    ctx.spmm(sg, dev(X), Y2, transpose=True, mask_bits=mb, Ylp=L2)
    assert torch.equal(Y1, Y2) and torch.equal(L1, L2)


@pytest.mark.parametrize("prec", [gsg.GSG_PREC_TF32, gsg.GSG_PREC_BF16])
@pytest.mark.parametrize("order2", [False, True])
def test_layer_bits_forward_and_backward(ctx, prec, order2):
    """layer_forward writes 1[H > 0] (GEMM epilogue in order 1, SpMM epilogue in order 2);
    layer_backward gated by those bits equals the call gated by the fp32 H_below."""
    g = graph(8000, 14.0, 1500, 120, 31)
    fi, fo = (300, 72) if order2 else (72, 300)
    rng = np.random.default_rng(32)
    X = rng.standard_normal((g.n, fi)).astype(np.float32)
    W = wl.glorot(rng, fi, fo)
    dH = rng.standard_normal((g.n, fo)).astype(np.float32)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    Xd, Wd = dev(X), dev(W)
    bf = prec == gsg.GSG_PREC_BF16
    Plp = torch.zeros((g.n, wl.ld_for(fi, 8)), dtype=torch.bfloat16, device="cuda")[:, :fi] if bf else None
    fl = gsg.GSG_ORDER_A_XW if order2 else 0
    P, H, Hb = empty(g.n, fo if order2 else fi), empty(g.n, fo), bits_buf(g.n, fo)
    ctx.layer_forward(sg, Xd, Wd, P, H, fi, fo, precision=prec, Plp=None if order2 else Plp, flags=fl, H_bits=Hb)
    assert np.array_equal(hbits(Hb), pack(h(H)))
    # the backward of a layer whose *input* was this H: gate its dX with H (bits vs fp32)
    if order2 and bf:
        ctx.to_bf16(Xd, Plp)
    # use (P, H) of this layer as the "below" gate source for a second layer of width fo -> fo
    W2 = wl.glorot(rng, fo, 40)
    W2d = dev(W2)
    P2, H2 = empty(g.n, fo), empty(g.n, 40)
    P2lp = torch.zeros((g.n, wl.ld_for(fo, 8)), dtype=torch.bfloat16, device="cuda")[:, :fo] if bf else None
    ctx.layer_forward(sg, H, W2d, P2, H2, fo, 40, precision=prec, Plp=P2lp)
    dH2 = dev(rng.standard_normal((g.n, 40)).astype(np.float32))
    outs = []
    for gate in ("fp32", "bits"):
        dW2, dX2 = empty(fo, 40), empty(g.n, fo)
        ctx.layer_backward(sg, P2, H2, dH2, W2d, dW2, dX2, fo, 40, precision=prec, Plp=P2lp,
                           H_below=H if gate == "fp32" else None, H_below_bits=Hb if gate == "bits" else None)
        outs.append((dW2, dX2))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    # order-2 backward (GEMM mask epilogue) of this layer, gated by an arbitrary below-mask
    Hbelow = rng.standard_normal((g.n, fi)).astype(np.float32)
    hbd, hbb = dev(Hbelow), torch.from_numpy(pack(Hbelow).view(np.int32)).cuda()
    outs = []
    for gate in ("fp32", "bits"):
        dW, dX = empty(fi, fo), empty(g.n, fi)
        ctx.layer_backward(sg, Xd if order2 else P, H, dev(dH), Wd, dW, dX, fi, fo, precision=prec, Plp=Plp,
                           H_below=hbd if gate == "fp32" else None, H_below_bits=hbb if gate == "bits" else None,
                           flags=fl)
        outs.append((dW, dX))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_head_bits(ctx):
    rng = np.random.default_rng(41)
    n, f, C = 1300, 200, 107
    HL = np.maximum(rng.standard_normal((n, f)), 0).astype(np.float32)
    Wm = wl.glorot(rng, f, C) * 8
    lab = torch.from_numpy((rng.random((n, C)) < 0.05).astype(np.uint8)).cuda()
    HLd, Wmd = dev(HL), dev(Wm)
    hb = torch.from_numpy(pack(HL).view(np.int32)).cuda()
    res = []
    for bits in (None, hb):
        S, dS, dWm, dHL = empty(n, C), empty(n, C), empty(f, C), empty(n, f)
        loss = torch.zeros(1, device="cuda")
        ctx.head(HLd, Wmd, lab, S, dS, dWm, dHL, n, f, C, gsg.GSG_HEAD_SIGMOID, loss, HL_bits=bits)
        res.append((dWm, dHL, loss))
    for a, b in zip(*res):
        assert torch.equal(a, b)


@pytest.mark.parametrize("cid", [2, 4])
def test_step_relu_bits_identical(ctx, cid):
    """A whole GCNStep (config 2: chain order 2 on layer 1, softmax head; config 4: BF16, 5 layers, no head)
    with bitmask gates gives bit-identical activations, gradients and loss to the fp32 gates."""
    cfg = wl.CONFIGS[cid]
    g = wl.sample_subgraph(cfg)
    inp = wl.make_inputs(cfg, g.n)
    sg = ctx.upload(g.indptr, g.indices)
    X = torch.zeros((g.n, wl.ld_for(cfg.dims[0])), device="cuda")[:, :cfg.dims[0]]
    X.copy_(torch.from_numpy(inp.X))
    labels = None if inp.labels is None else torch.from_numpy(inp.labels).cuda()
    dH = None
    if inp.dH is not None:
        dH = torch.zeros((g.n, wl.ld_for(cfg.dims[-1])), device="cuda")[:, :cfg.dims[-1]]
        dH.copy_(torch.from_numpy(inp.dH))
    res = []
    for rb in (False, True):
        step = GCNStep(ctx, cfg.dims, g.n, cfg.head, cfg.classes, cfg.precision, weights=inp.Ws, w_mlp=inp.W_mlp,
                       relu_bits=rb)
        step.forward_backward(sg, X, labels=labels, dH_top=dH)
        ctx.sync()
        res.append([t.clone() for t in step.H + step.dX] + [step.grad_flat.clone(), step.loss.clone()])
    for a, b in zip(*res):
        assert torch.equal(a, b)


def test_bits_argument_errors(ctx):
    g = graph(2000, 8.0, 300, 30, 3)
    sg = ctx.upload(g.indptr, g.indices).normalize()
    X, W = dev(np.ones((g.n, 40))), dev(np.ones((40, 70)))
    with pytest.raises(gsg.GsgError) as e:      # bits need the ReLU epilogue
        ctx.layer_forward(sg, X, W, empty(g.n, 40), empty(g.n, 70), 40, 70, flags=gsg.GSG_NO_RELU,
                          H_bits=bits_buf(g.n, 70))
    assert e.value.code == gsg.GSG_EINVAL
    with pytest.raises(gsg.GsgError) as e:      # ld below ceil(f/32) words
        ctx.gemm(X, W, empty(g.n, 70), epilogue=gsg.GSG_EPI_RELU, C_bits=bits_buf(g.n, 40, pad=0))
    assert e.value.code == gsg.GSG_EINVAL
    with pytest.raises(gsg.GsgError) as e:      # gate bits with a non-mask epilogue
        ctx.gemm(X, W, empty(g.n, 70), aux_bits=bits_buf(g.n, 70))
    assert e.value.code == gsg.GSG_EINVAL
