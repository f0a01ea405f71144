"""GSG_PREC_FP32X3 (3xTF32, gsg.h): fp32-accurate GEMMs on the TF32 tensor cores, the precision
configs 1-2 ("fp32" in BASELINE.json) run in. Graded at the fp32 SpMM tolerance, 1e-5
(max-normalized, against the fp64 oracle), for every operand majorness, split-K, every
epilogue, the layer calls (stage-isolated) and the head; and shown to be far more accurate
than plain TF32 on the same inputs (so the split path is really taken)."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2010_03166_b200 as gsg
import workload as wl
from test_gpu_parity import dev, empty, host, rel_err

pytestmark = pytest.mark.gpu

X3_TOL = 1e-5
X3 = gsg.GSG_PREC_FP32X3


@pytest.fixture(scope="module")
def ctx():
    c = gsg.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 200, 50), (1000, 512, 602), (130, 17, 5), (602, 512, 3000),
                                   (50, 128, 2000), (2000, 41, 512)])
def test_gemm_fp32x3_vs_oracle(ctx, ta, tb, M, N, K):
    rng = np.random.default_rng(M * 5 + N * 11 + K)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = orc.gemm(A, B, ta, tb)
    C, Ct = empty(M, N), empty(M, N)
    ctx.gemm(dev(A), dev(B), C, transA=ta, transB=tb, precision=X3, K=K)
    ctx.gemm(dev(A), dev(B), Ct, transA=ta, transB=tb, precision=gsg.GSG_PREC_TF32, K=K)
    e3, e1 = rel_err(host(C), ref), rel_err(host(Ct), ref)
    assert e3 <= X3_TOL, e3
    assert e3 < e1 / 20, (e3, e1)  # the split path, not plain TF32


@pytest.mark.parametrize("split", [1, 3, 16])
def test_gemm_fp32x3_epilogues_splitk(ctx, split):
    """ReLU (+ bitmask, bf16 copy), ReLU' gate (fp32 and bitmask), accumulate; forced K splits
    (the dW shape: MN-major operands, K = n); deterministic. (A caller-forced split count is
    honoured as given, so the pieces here stay at K' <= 1200: the tensor-core accumulator, not the
    split, bounds the accuracy of one long K piece -- 1.5e-5 at K' = 3600; the automatic split
    keeps pieces at K' <= 1024, see test_gemm_fp32x3_long_k_auto_split.)"""
    rng = np.random.default_rng(split)
    M, N, K = 300, 200, (300 if split == 1 else 1200)  # a forced single piece: K' = 900
    A = rng.standard_normal((K, M)).astype(np.float32)  # stored K x M (transA)
    B = rng.standard_normal((K, N)).astype(np.float32)
    aux = rng.standard_normal((M, N)).astype(np.float32)
    ref = orc.gemm(A, B, True, False)
    C = empty(M, N)
    ctx.gemm(dev(A), dev(B), C, transA=True, precision=X3, epilogue=gsg.GSG_EPI_MASK, aux=dev(aux), split_k=split, K=K)
    assert rel_err(host(C), np.where(aux > 0, ref, 0)) <= X3_TOL
    C2 = empty(M, N)
    ctx.gemm(dev(A), dev(B), C2, transA=True, precision=X3, epilogue=gsg.GSG_EPI_MASK, aux=dev(aux), split_k=split, K=K)
    assert torch.equal(C, C2)
    Cd = dev(np.ones((M, N), np.float32))
    ctx.gemm(dev(A), dev(B), Cd, transA=True, precision=X3, accumulate=True, split_k=split, K=K)
    assert rel_err(host(Cd), ref + 1.0) <= X3_TOL
    # ReLU with the bitmask output (forces one split) and the bf16 copy
    Cr = empty(M, N)
    bits = torch.zeros((M, (N + 31) // 32), dtype=torch.int32, device="cuda")
    Clp = torch.zeros((M, wl.ld_for(N, 8)), dtype=torch.bfloat16, device="cuda")[:, :N]
    ctx.gemm(dev(A), dev(B), Cr, transA=True, precision=X3, epilogue=gsg.GSG_EPI_RELU, Clp=Clp, C_bits=bits, K=K)
    assert rel_err(host(Cr), np.maximum(ref, 0)) <= X3_TOL
    hb = bits.cpu().numpy().view(np.uint32)
    got = ((hb[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(M, -1)[:, :N]
    assert np.array_equal(got.astype(bool), host(Cr) > 0)
    # ReLU' gate from the bitmask
    Cg = empty(M, N)
    ctx.gemm(dev(A), dev(B), Cg, transA=True, precision=X3, epilogue=gsg.GSG_EPI_MASK, aux_bits=bits, K=K)
    assert rel_err(host(Cg), np.where(host(Cr) > 0, ref, 0)) <= X3_TOL


def test_layer_fp32x3_stage_isolated(ctx):
    """Config 1's layer (50 -> 128) through gsg_layer_forward / gsg_layer_backward in FP32X3:
    every stage at 1e-5 (the SpMMs are fp32 anyway; the GEMMs now match them)."""
    cfg = wl.CONFIGS[1]
    g = wl.sample_subgraph(cfg)
    inp = wl.make_inputs(cfg, g.n)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    n, fi, fo = g.n, 50, 128
    sg = ctx.upload(g.indptr, g.indices).normalize()
    Hb = np.random.default_rng(3).standard_normal((n, fi)).astype(np.float32)
    Wd = dev(inp.Ws[0])
    P, H = empty(n, fi), empty(n, fo)
    ctx.layer_forward(sg, dev(inp.X), Wd, P, H, fi, fo, precision=X3)
    dW, dX = empty(fi, fo), empty(n, fi)
    ctx.layer_backward(sg, P, H, dev(inp.dH), Wd, dW, dX, fi, fo, precision=X3, H_below=dev(Hb))
    Pg, Hg = host(P), host(H)
    assert rel_err(Pg, orc.spmm(A, inp.X)) <= X3_TOL
    assert rel_err(Hg, np.maximum(orc.gemm(Pg, inp.Ws[0]), 0)) <= X3_TOL
    dZ = orc.relu_mask(inp.dH, Hg)
    assert rel_err(host(dW), orc.gemm(Pg, dZ, transA=True)) <= X3_TOL
    T = orc.gemm(dZ, inp.Ws[0], transB=True)
    assert rel_err(host(dX), np.where(Hb > 0, orc.spmm_t(A, T), 0)) <= X3_TOL


@pytest.mark.parametrize("kind,C", [("softmax", 41), ("sigmoid", 107)])
def test_head_fp32x3(ctx, kind, C):
    rng = np.random.default_rng(18)
    n, f = 1200, 512
    HL = np.maximum(rng.standard_normal((n, f)), 0).astype(np.float32)
    Wm = wl.glorot(rng, f, C) * 8
    labels = rng.integers(0, C, n).astype(np.int32) if kind == "softmax" else (rng.random((n, C)) < 0.05).astype(np.uint8)
    S = empty(n, C)
    dS = torch.full((n, S.stride(0)), float("nan"), device="cuda")[:, :C]
    dWm, dHL = empty(f, C), empty(n, f)
    loss = torch.zeros(1, device="cuda")
    ctx.head(dev(HL), dev(Wm), torch.from_numpy(labels).cuda(), S, dS, dWm, dHL, n, f, C,
             gsg.GSG_HEAD_SOFTMAX if kind == "softmax" else gsg.GSG_HEAD_SIGMOID, loss, precision=X3)
    Sg = host(S)
    assert rel_err(Sg, orc.gemm(HL, Wm)) <= X3_TOL
    dSg = host(dS)
    _, _, dS_ref = orc.head(Sg, labels, kind)
    assert rel_err(dSg, dS_ref) <= 1e-5
    assert rel_err(host(dWm), orc.gemm(HL, dSg, transA=True)) <= X3_TOL
    assert rel_err(host(dHL), np.where(HL > 0, orc.gemm(dSg, Wm, transB=True), 0)) <= X3_TOL


@pytest.mark.parametrize("ta", [True, False])
def test_gemm_fp32x3_long_k_auto_split(ctx, ta):
    """K = 20000 (config 5's dW contraction length): the automatic split keeps every K piece
    short enough (K' <= 4096) for 1e-5, also where the tile count alone would not split."""
    rng = np.random.default_rng(7)
    M, N, K = 1024, 1024, 20000
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((K, N)).astype(np.float32)
    C = empty(M, N)
    ctx.gemm(dev(A), dev(B), C, transA=ta, precision=X3, K=K)
    rows = np.arange(0, M, 37)
    ref = orc.gemm(A[:, rows].T if ta else A[rows], B)
    assert rel_err(host(C)[rows], ref) <= X3_TOL


def test_tf32_operand_is_truncated(ctx):
    """The premise of FP32X3's implicit hi (gemm.cu k_split_lo): kind::tf32 reads an fp32 operand
    by truncating it to tf32, so the unmodified operand is hi = trunc(x) and lo = x - trunc(x).
    A single product 1 x (1 + 0.75 / 0.5 / 0.25 ulp_tf32) must come out as exactly 1 (rounding to
    nearest would give 1 + ulp for 0.75); the negative case truncates toward zero."""
    M = N = 128
    K = 32
    for v in (1 + 2**-11 + 2**-12, 1 + 2**-11, 1 + 2**-12, -(1 + 2**-11 + 2**-12)):
        A = np.zeros((M, K), np.float32)
        A[:, 0] = v
        B = np.zeros((K, N), np.float32)
        B[0, :] = 1.0
        C = empty(M, N)
        ctx.gemm(dev(A), dev(B), C, precision=gsg.GSG_PREC_TF32, K=K)
        assert np.all(host(C) == np.float32(1.0 if v > 0 else -1.0)), (v, host(C)[0, 0])



@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_gemm_fp32x3_unaligned_strides(ctx, ta, tb):
    """FP32X3 takes operands whose row pitch TMA cannot read in place (ld % 4 != 0): the split
    also copies them (implicit hi), same 1e-5."""
    rng = np.random.default_rng(5)
    M, N, K = 300, 130, 602
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    ref = orc.gemm(A, B, ta, tb)
    C = empty(M, N)
    ctx.gemm(dev(A, ld=A.shape[1] + 1), dev(B, ld=B.shape[1] + 2), C, transA=ta, transB=tb, precision=X3, K=K)
    assert rel_err(host(C), ref) <= X3_TOL
