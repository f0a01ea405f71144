"""Every output element of the big GEMMs at the benchmark configs' own shapes against the fp64
oracle (SURVEY §8(c) stage isolation; the full-size step tests in test_gpu_fullsize.py sample
rows): config 5's Z = P·W with the ReLU / bitmask / bf16 epilogue, T = dZ·Wᵀ and the split-K
dW = Pᵀ·dZ (K = 20,000) in TF32; config 4's in BF16; config 2's FP32X3 GEMMs (1e-5), including
its dW (K = 8,000, split over CTAs and over the two TMEM halves of a tile).
Operands are N(0, 1) (P, dZ) and Glorot-scaled (W) like the step's; max-normalized error."""
import numpy as np
import pytest
import torch

import oracle as orc
import paper_2010_03166_b200 as gsg
import workload as wl
from test_gpu_parity import GEMM_TOL, dev, empty, host, rel_err

pytestmark = pytest.mark.gpu

X3_TOL = 1e-5


@pytest.fixture(scope="module")
def ctx():
    c = gsg.Context(0)
    yield c
    c.close()


def _bf16(a: np.ndarray):
    """bf16 device copy (row stride a multiple of 8) and the fp32 values it holds."""
    t = torch.zeros((a.shape[0], wl.ld_for(a.shape[1], 8)), dtype=torch.bfloat16, device="cuda")[:, :a.shape[1]]
    t.copy_(torch.from_numpy(a))
    return t, t.float().cpu().numpy()


@pytest.mark.parametrize("n,f", [(20000, 1024)])
def test_tf32_forward_full(ctx, n, f):
    rng = np.random.default_rng(51)
    P = rng.standard_normal((n, f)).astype(np.float32)
    W = wl.glorot(rng, f, f)
    Z = orc.gemm(P, W)
    C = empty(n, f)
    bits = torch.zeros((n, f // 32), dtype=torch.int32, device="cuda")
    Clp = torch.zeros((n, wl.ld_for(f, 8)), dtype=torch.bfloat16, device="cuda")[:, :f]
    ctx.gemm(dev(P), dev(W), C, epilogue=gsg.GSG_EPI_RELU, Clp=Clp, C_bits=bits)
    H = host(C)
    assert rel_err(H, np.maximum(Z, 0)) <= GEMM_TOL
    hb = bits.cpu().numpy().view(np.uint32)
    got = ((hb[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(n, -1)[:, :f].astype(bool)
    assert np.array_equal(got, H > 0)
    assert np.array_equal(Clp.float().cpu().numpy(), torch.from_numpy(H).to(torch.bfloat16).float().numpy())


@pytest.mark.parametrize("n,f_in,f_out", [(20000, 1024, 1024)])
def test_tf32_backward_full(ctx, n, f_in, f_out):
    rng = np.random.default_rng(52)
    P = rng.standard_normal((n, f_in)).astype(np.float32)
    dZ = rng.standard_normal((n, f_out)).astype(np.float32)
    W = wl.glorot(rng, f_in, f_out)
    T = empty(n, f_in)
    ctx.gemm(dev(dZ), dev(W), T, transB=True)  # T = dZ Wᵀ
    assert rel_err(host(T), orc.gemm(dZ, W, False, True)) <= GEMM_TOL
    dW = empty(f_in, f_out)
    ctx.gemm(dev(P), dev(dZ), dW, transA=True)  # dW = Pᵀ dZ, split-K (K = n)
    assert rel_err(host(dW), orc.gemm(P, dZ, True, False)) <= GEMM_TOL


@pytest.mark.parametrize("n,f", [(16000, 1024)])
def test_bf16_full(ctx, n, f):
    rng = np.random.default_rng(53)
    P, Pv = _bf16(rng.standard_normal((n, f)).astype(np.float32))
    W, Wv = _bf16(wl.glorot(rng, f, f))
    dZ, dZv = _bf16(rng.standard_normal((n, f)).astype(np.float32))
    C = empty(n, f)
    ctx.gemm(P, W, C, precision=gsg.GSG_PREC_BF16)
    assert rel_err(host(C), orc.gemm(Pv, Wv)) <= GEMM_TOL
    dW = empty(f, f)
    ctx.gemm(P, dZ, dW, transA=True, precision=gsg.GSG_PREC_BF16)
    assert rel_err(host(dW), orc.gemm(Pv, dZv, True, False)) <= GEMM_TOL


@pytest.mark.parametrize("n,f_in,f_out", [(8000, 602, 512)])
def test_fp32x3_full(ctx, n, f_in, f_out):
    rng = np.random.default_rng(54)
    P = rng.standard_normal((n, f_in)).astype(np.float32)
    W = wl.glorot(rng, f_in, f_out)
    dZ = rng.standard_normal((n, f_out)).astype(np.float32)
    X3 = gsg.GSG_PREC_FP32X3
    Z = empty(n, f_out)
    ctx.gemm(dev(P), dev(W), Z, precision=X3)  # K = 602: one CTA, two TMEM halves per tile
    assert rel_err(host(Z), orc.gemm(P, W)) <= X3_TOL
    T = empty(n, f_in)
    ctx.gemm(dev(dZ), dev(W), T, transB=True, precision=X3)
    assert rel_err(host(T), orc.gemm(dZ, W, False, True)) <= X3_TOL
    dW = empty(f_in, f_out)
    ctx.gemm(dev(P), dev(dZ), dW, transA=True, precision=X3)  # K = 8000: split over CTAs too
    assert rel_err(host(dW), orc.gemm(P, dZ, True, False)) <= X3_TOL
