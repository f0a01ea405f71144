"""Pins for the fp64 oracle (oracle/), independent of the oracle's own code.

Each test ties an oracle function to something other than itself (SURVEY §8(c) "What pins
each part"): hand-derived closed forms (golden fixtures), SPEC examples, dense brute force
with numpy's own matmul, the adjoint identity, central finite differences and structural
invariants. A dropped term, a wrong sign or index, or a transposed operand in any oracle
function fails at least one of these.
"""
import json
import os

import numpy as np
import pytest
from scipy.special import logsumexp

import oracle as orc
import workload as wl

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rand_graph(n, deg, seed):
    p = wl.Parent(n, deg, 2.1, 0.0, seed=seed)
    return p.csr()


def dense_adj(csr):
    A = np.zeros((csr.n, csr.n))
    for i in range(csr.n):
        A[i, csr.indices[csr.indptr[i]:csr.indptr[i + 1]]] = 1.0
    return A


# ------------------------------------------------------------------------------ Â (a1)
def test_golden_p3_row_self():
    g = load("p3_path.json")
    A = orc.normalize(g["graph"]["indptr"], g["graph"]["indices"], orc.NORM_ROW_SELF)
    np.testing.assert_allclose(A.dense(), g["A_hat_row_self"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(A.dense().sum(0), g["column_sums"], rtol=0, atol=1e-15)
    vt = orc.transpose_alg4(A)
    AT = orc.AHat(A.indptr, A.idx, vt).dense()
    np.testing.assert_allclose(AT, g["A_hat_row_self_T"], rtol=0, atol=1e-15)
    # self loops are inserted at the sorted position: row 1 = [0, 1, 2]
    assert list(A.idx[A.indptr[1]:A.indptr[2]]) == [0, 1, 2]


def test_golden_sym_p2():
    g = load("sym_p2.json")
    A = orc.normalize(g["graph"]["indptr"], g["graph"]["indices"], orc.NORM_SYM_SELF)
    np.testing.assert_allclose(A.dense(), g["A_hat_sym_self"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("mode", [orc.NORM_ROW_SELF, orc.NORM_SYM_SELF])
def test_no_edges_is_identity(mode):
    A = orc.normalize(np.zeros(6, np.int64), np.zeros(0, np.int32), mode)
    np.testing.assert_array_equal(A.dense(), np.eye(5))


@pytest.mark.parametrize("mode", [orc.NORM_ROW_SELF, orc.NORM_SYM_SELF])
def test_complete_graph_is_J_over_n(mode):
    n = 7
    ip = np.arange(0, n * (n - 1) + 1, n - 1, dtype=np.int64)
    ix = np.array([j for i in range(n) for j in range(n) if j != i], np.int32)
    A = orc.normalize(ip, ix, mode)
    np.testing.assert_allclose(A.dense(), np.full((n, n), 1.0 / n), rtol=0, atol=1e-15)


def test_row_modes_match_dense_definition():
    g = rand_graph(60, 6.0, 1)
    Ad = dense_adj(g)
    d = Ad.sum(1)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    np.testing.assert_allclose(A.dense(), np.diag(1 / (d + 1)) @ (Ad + np.eye(g.n)), atol=1e-15)
    np.testing.assert_allclose(A.dense().sum(1), 1.0, atol=1e-15)  # row-stochastic
    S = orc.normalize(g.indptr, g.indices, orc.NORM_SYM_SELF)
    Dm = np.diag(1 / np.sqrt(d + 1))
    np.testing.assert_allclose(S.dense(), Dm @ (Ad + np.eye(g.n)) @ Dm, atol=1e-15)  # Eq. 5
    R = orc.normalize(g.indptr, g.indices, orc.NORM_ROW)
    Dinv = np.diag(np.where(d > 0, 1 / np.maximum(d, 1), 0))
    np.testing.assert_allclose(R.dense(), Dinv @ Ad, atol=1e-15)  # GraphSAGE Eq. 1
    nz = d > 0
    np.testing.assert_allclose(R.dense().sum(1)[nz], 1.0, atol=1e-15)


def test_values_mode_is_the_given_matrix():
    """GSG_NORM_VALUES (weighted Â): Â_ij = value of the stored edge (i, j) and no
    self loop. Pinned against a dense matrix built here directly from (indptr, indices, values)
    by numpy fancy indexing -- not through AHat.dense() -- and through the products: ÂX and ÂᵀT
    with numpy's matmul of that matrix (values deliberately asymmetric: v(i,j) != v(j,i))."""
    g = rand_graph(70, 6.0, 21)
    rng = np.random.default_rng(22)
    vals = rng.uniform(-1.0, 2.0, g.nnz)
    rows = np.repeat(np.arange(g.n), np.diff(g.indptr))
    D = np.zeros((g.n, g.n))
    D[rows, g.indices] = vals
    assert not np.allclose(D, D.T)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_VALUES, vals)
    np.testing.assert_array_equal(A.indptr, g.indptr)
    np.testing.assert_array_equal(A.idx, g.indices)
    np.testing.assert_array_equal(A.val, vals)
    np.testing.assert_array_equal(A.dense(), D)
    X = rng.standard_normal((g.n, 5))
    np.testing.assert_allclose(orc.spmm(A, X), D @ X, rtol=0, atol=1e-12)
    np.testing.assert_allclose(orc.spmm_t(A, X), D.T @ X, rtol=0, atol=1e-12)
    vt = orc.transpose_alg4(A)
    DT = np.zeros((g.n, g.n))
    DT[rows, g.indices] = vt
    np.testing.assert_array_equal(DT, D.T)


# ------------------------------------------------------------------------------ Alg. 4
def test_alg4_two_node_swap():
    # data for (0,1)=x, (1,0)=y -> transposed data has y at (0,1)'s slot
    A = orc.AHat(np.array([0, 1, 2], np.int64), np.array([1, 0], np.int32), np.array([3.0, 5.0]))
    np.testing.assert_array_equal(orc.transpose_alg4(A), [5.0, 3.0])


def test_alg4_equals_dense_transpose_and_involution():
    g = rand_graph(80, 7.0, 2)
    vals = np.random.default_rng(3).uniform(0.1, 1.0, g.nnz)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_VALUES, vals)
    vt = orc.transpose_alg4(A)
    np.testing.assert_array_equal(orc.AHat(A.indptr, A.idx, vt).dense(), A.dense().T)
    vtt = orc.transpose_alg4(orc.AHat(A.indptr, A.idx, vt))
    np.testing.assert_array_equal(vtt, A.val)  # involution


def test_alg4_symmetric_fixed_point():
    g = rand_graph(50, 5.0, 4)
    S = orc.normalize(g.indptr, g.indices, orc.NORM_SYM_SELF)
    np.testing.assert_array_equal(orc.transpose_alg4(S), S.val)


def test_alg4_row_mode_closed_form():
    # Âᵀ_uv = Â_vu = 1/(d_v+1) in row mode
    g = rand_graph(70, 6.0, 5)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    vt = orc.transpose_alg4(A)
    d = np.diff(g.indptr).astype(np.float64)
    np.testing.assert_array_equal(vt, 1.0 / (d[A.idx] + 1.0))


# ------------------------------------------------------------------------------ SpMM (a2, a7)
@pytest.mark.parametrize("n,deg,f,seed", [(40, 5.0, 3, 6), (64, 9.0, 17, 7), (30, 3.0, 1, 8)])
def test_spmm_dense_bruteforce(n, deg, f, seed):
    g = rand_graph(n, deg, seed)
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((g.n, f))
    for mode in (orc.NORM_ROW_SELF, orc.NORM_SYM_SELF, orc.NORM_ROW):
        A = orc.normalize(g.indptr, g.indices, mode)
        Ad = A.dense()
        np.testing.assert_allclose(orc.spmm(A, X), Ad @ X, rtol=1e-13, atol=1e-13)
        T = rng.standard_normal((g.n, f))
        np.testing.assert_allclose(orc.spmm_t(A, T), Ad.T @ T, rtol=1e-13, atol=1e-13)


def test_spmm_special_cases():
    g = rand_graph(50, 6.0, 9)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    np.testing.assert_allclose(orc.spmm(A, np.ones((g.n, 4))), 1.0, atol=1e-14)
    I = orc.normalize(np.zeros(11, np.int64), np.zeros(0, np.int32), orc.NORM_ROW_SELF)
    X = np.random.default_rng(0).standard_normal((10, 5))
    np.testing.assert_array_equal(orc.spmm(I, X), X)  # Â = I -> P = X
    n = 6
    ip = np.arange(0, n * (n - 1) + 1, n - 1, dtype=np.int64)
    ix = np.array([j for i in range(n) for j in range(n) if j != i], np.int32)
    K = orc.normalize(ip, ix, orc.NORM_ROW_SELF)
    Xk = np.random.default_rng(1).standard_normal((n, 3))
    np.testing.assert_allclose(orc.spmm(K, Xk), np.tile(Xk.mean(0), (n, 1)), atol=1e-15)


def test_adjoint_identity():
    """<Â X, G> = <X, Âᵀ G> pins the scatter-form transpose against the gather-form SpMM."""
    g = rand_graph(500, 12.0, 10)
    rng = np.random.default_rng(11)
    vals = rng.uniform(0.1, 1.0, g.nnz)
    for A in (orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF),
              orc.normalize(g.indptr, g.indices, orc.NORM_VALUES, vals)):
        X = rng.standard_normal((g.n, 9))
        G = rng.standard_normal((g.n, 9))
        lhs = np.sum(orc.spmm(A, X) * G)
        rhs = np.sum(X * orc.spmm_t(A, G))
        assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


def test_scatter_transpose_equals_gather_over_alg4():
    g = rand_graph(300, 10.0, 12)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_VALUES,
                      np.random.default_rng(13).uniform(0.1, 1.0, g.nnz))
    AT = orc.AHat(A.indptr, A.idx, orc.transpose_alg4(A))
    T = np.random.default_rng(14).standard_normal((g.n, 6))
    np.testing.assert_allclose(orc.spmm_t(A, T), orc.spmm(AT, T), rtol=1e-13, atol=1e-13)


def test_row_range():
    g = rand_graph(90, 6.0, 15)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    X = np.random.default_rng(16).standard_normal((g.n, 5))
    full = orc.spmm(A, X)
    part = orc.spmm(A, X, 10, 40)
    np.testing.assert_array_equal(part[10:40], full[10:40])
    assert not part[:10].any() and not part[40:].any()
    a = orc.spmm_t(A, X, 0, 45) + orc.spmm_t(A, X, 45, g.n)
    np.testing.assert_allclose(a, orc.spmm_t(A, X), atol=1e-14)


# ------------------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_vs_numpy(ta, tb):
    rng = np.random.default_rng(17)
    M, N, K = 13, 9, 21
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    ref = (A.T if ta else A) @ (B.T if tb else B)
    np.testing.assert_allclose(orc.gemm(A, B, ta, tb), ref, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------------------ layer
def test_layer_forward_special_cases():
    g = rand_graph(40, 5.0, 18)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    rng = np.random.default_rng(19)
    W = rng.standard_normal((6, 4))
    _, _, H = orc.layer_forward(A, np.zeros((g.n, 6)), W)
    assert not H.any()
    Xp = np.abs(rng.standard_normal((g.n, 6)))
    _, _, H = orc.layer_forward(A, Xp, np.eye(6))
    np.testing.assert_allclose(H, A.dense() @ Xp, atol=1e-14)
    I = orc.normalize(np.zeros(g.n + 1, np.int64), np.zeros(0, np.int32), orc.NORM_ROW_SELF)
    X = rng.standard_normal((g.n, 6))
    _, _, H = orc.layer_forward(I, X, W)
    np.testing.assert_allclose(H, np.maximum(X @ W, 0), atol=1e-14)


def test_mask_semantics():
    Z = np.array([[1.0, -1.0, 0.0], [-0.0, 2.0, -3.0]])
    dH = np.array([[5.0, 6.0, 7.0], [8.0, 9.0, 10.0]])
    np.testing.assert_array_equal(orc.relu_mask(dH, Z), [[5.0, 0, 0], [0, 9.0, 0]])  # ReLU'(0)=0


def _fd_check(fun, x, grad, coords, h=1e-6, sign_fun=None, tol=1e-6):
    checked = 0
    for c in coords:
        xp = x.copy(); xp[c] += h
        xm = x.copy(); xm[c] -= h
        if sign_fun is not None and not np.array_equal(sign_fun(xp), sign_fun(xm)):
            continue  # a ReLU kink lies inside the stencil
        fd = (fun(xp) - fun(xm)) / (2 * h)
        assert abs(fd - grad[c]) <= tol * max(1.0, abs(fd)), (c, fd, grad[c])
        checked += 1
    assert checked >= len(coords) // 2


def test_layer_backward_finite_differences():
    """Central FD of the probe loss <H, dH> w.r.t. W and X (SURVEY §8(c) pin for a4-a7)."""
    g = rand_graph(30, 5.0, 20)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_SYM_SELF)  # asymmetric-free but non-uniform
    Av = orc.normalize(g.indptr, g.indices, orc.NORM_VALUES,
                       np.random.default_rng(21).uniform(0.1, 1.0, g.nnz))  # nonsymmetric Â
    rng = np.random.default_rng(22)
    for Ah in (A, Av):
        X = rng.standard_normal((g.n, 5))
        W = rng.standard_normal((5, 4))
        dH = rng.standard_normal((g.n, 4))
        P, Z, H = orc.layer_forward(Ah, X, W)
        _, dW, _, dX = orc.layer_backward(Ah, P, Z, dH, W)
        lossW = lambda w: float(np.sum(orc.layer_forward(Ah, X, w)[2] * dH))
        lossX = lambda x: float(np.sum(orc.layer_forward(Ah, x, W)[2] * dH))
        signW = lambda w: orc.layer_forward(Ah, X, w)[1] > 0
        signX = lambda x: orc.layer_forward(Ah, x, W)[1] > 0
        coordsW = [(i, j) for i in range(5) for j in range(4)]
        coordsX = [(int(i), int(j)) for i, j in zip(rng.integers(0, g.n, 25), rng.integers(0, 5, 25))]
        _fd_check(lossW, W, dW, coordsW, sign_fun=signW)
        _fd_check(lossX, X, dX, coordsX, sign_fun=signX)


@pytest.mark.parametrize("kind,C", [("softmax", 5), ("sigmoid", 6)])
def test_model_finite_differences(kind, C):
    """FD through a 2-layer GCN + ReLU/softmax|sigmoid head (Eqs. 2-4, 9-15)."""
    g = rand_graph(25, 5.0, 23)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    rng = np.random.default_rng(24)
    X = rng.standard_normal((g.n, 4))
    Ws = [rng.standard_normal((4, 5)), rng.standard_normal((5, 3))]
    Wm = rng.standard_normal((3, C))
    labels = rng.integers(0, C, g.n).astype(np.int32) if kind == "softmax" else \
        (rng.random((g.n, C)) < 0.3).astype(np.uint8)
    out = orc.model_step(A, X, Ws, Wm, labels, kind)

    def loss_of(ws, wm):
        return orc.model_step(A, X, ws, wm, labels, kind)["loss"]

    def signs(ws, wm):
        o = orc.model_step(A, X, ws, wm, labels, kind)
        return np.concatenate([z.ravel() > 0 for z in o["Z"]] + [o["S"].ravel() > 0])

    coords = [(i, j) for i in range(4) for j in range(5)]
    _fd_check(lambda w: loss_of([w, Ws[1]], Wm), Ws[0], out["dW"][0], coords,
              sign_fun=lambda w: signs([w, Ws[1]], Wm))
    coords = [(i, j) for i in range(3) for j in range(C)]
    _fd_check(lambda w: loss_of(Ws, w), Wm, out["dW_mlp"], coords, sign_fun=lambda w: signs(Ws, w))


def test_sage_forward_special_cases_and_dense():
    """GraphSAGE (Eq. 1): an isolated node's neighbor half is 0 (Ã row = 0, SPEC S:120
    design decision); W_s = W_n = I with X >= 0 gives [X | ÃX]; dense D⁻¹A brute force."""
    g = rand_graph(50, 4.0, 30)
    ip = np.concatenate([g.indptr, [g.indptr[-1]]]).astype(np.int64)   # append an isolated node
    A = orc.normalize(ip, g.indices, orc.NORM_ROW)
    n = g.n + 1
    rng = np.random.default_rng(31)
    Xp = np.abs(rng.standard_normal((n, 6)))
    _, _, H = orc.sage_forward(A, Xp, np.eye(6), np.eye(6))
    Ad = dense_adj(wl.CSR(ip, g.indices))
    d = Ad.sum(1)
    Abar = np.diag(np.where(d > 0, 1 / np.maximum(d, 1), 0)) @ Ad
    np.testing.assert_allclose(H, np.hstack([Xp, Abar @ Xp]), atol=1e-14)
    assert not H[-1, 6:].any()
    X = rng.standard_normal((n, 6))
    Ws, Wn = rng.standard_normal((6, 4)), rng.standard_normal((6, 4))
    _, Z, H = orc.sage_forward(A, X, Ws, Wn)
    np.testing.assert_allclose(Z, np.hstack([X @ Ws, Abar @ X @ Wn]), rtol=1e-13, atol=1e-13)


def test_sage_backward_finite_differences():
    """Eqs. 12-15 against central differences of <H, dH> w.r.t. W_s, W_n and X."""
    g = rand_graph(30, 5.0, 32)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW)
    rng = np.random.default_rng(33)
    X = rng.standard_normal((g.n, 5))
    Ws, Wn = rng.standard_normal((5, 3)), rng.standard_normal((5, 3))
    dH = rng.standard_normal((g.n, 6))
    P, Z, H = orc.sage_forward(A, X, Ws, Wn)
    _, dWs, dWn, dX = orc.sage_backward(A, X, P, Z, dH, Ws, Wn)
    loss = lambda x, ws, wn: float(np.sum(orc.sage_forward(A, x, ws, wn)[2] * dH))
    sign = lambda x, ws, wn: orc.sage_forward(A, x, ws, wn)[1] > 0
    cw = [(i, j) for i in range(5) for j in range(3)]
    _fd_check(lambda w: loss(X, w, Wn), Ws, dWs, cw, sign_fun=lambda w: sign(X, w, Wn))
    _fd_check(lambda w: loss(X, Ws, w), Wn, dWn, cw, sign_fun=lambda w: sign(X, Ws, w))
    cx = [(int(i), int(j)) for i, j in zip(rng.integers(0, g.n, 20), rng.integers(0, 5, 20))]
    _fd_check(lambda x: loss(x, Ws, Wn), X, dX, cx, sign_fun=lambda x: sign(x, Ws, Wn))


def test_head_closed_forms():
    n, C = 8, 41
    loss, Y, dS = orc.head(np.zeros((n, C)), np.zeros(n, np.int32), "softmax")
    assert abs(loss - np.log(C)) < 1e-14  # uniform softmax -> ln C
    np.testing.assert_allclose(Y.sum(1), 1.0, atol=1e-15)
    assert not dS.any()  # S = 0 -> ReLU mask kills every gradient entry (Eq. 10 mask)
    loss, Y, _ = orc.head(np.zeros((n, 7)), np.zeros((n, 7), np.uint8), "sigmoid")
    assert abs(loss - 7 * np.log(2.0)) < 1e-13


def test_head_vs_library_formulas():
    rng = np.random.default_rng(25)
    n, C = 20, 9
    S = rng.standard_normal((n, C))
    Sp = np.maximum(S, 0)
    y = rng.integers(0, C, n).astype(np.int32)
    loss, Y, dS = orc.head(S, y, "softmax")
    ref = -np.mean(Sp[np.arange(n), y] - logsumexp(Sp, axis=1))
    assert abs(loss - ref) < 1e-13
    Ybar = np.eye(C)[y]
    np.testing.assert_allclose(dS, (Y - Ybar) / n * (S > 0), atol=1e-15)  # P:689 + Eq. 10 mask
    yb = (rng.random((n, C)) < 0.4).astype(np.uint8)
    loss, Y, dS = orc.head(S, yb, "sigmoid")
    sig = 1 / (1 + np.exp(-Sp))
    ref = -np.mean(np.sum(yb * np.log(sig) + (1 - yb) * np.log(1 - sig), axis=1))
    assert abs(loss - ref) < 1e-12
    np.testing.assert_allclose(dS, (sig - yb) / n * (S > 0), atol=1e-15)


def test_head_node_weights():
    """GraphSAINT loss normalization: weighted sum of per-node CE; λ = 1/n is the mean."""
    rng = np.random.default_rng(40)
    n, C = 16, 5
    S = rng.standard_normal((n, C))
    y = rng.integers(0, C, n).astype(np.int32)
    l0, _, g0 = orc.head(S, y, "softmax")
    l1, _, g1 = orc.head(S, y, "softmax", np.full(n, 1.0 / n))
    assert abs(l0 - l1) < 1e-15 and np.allclose(g0, g1, rtol=0, atol=1e-17)
    lam = rng.uniform(0.01, 0.2, n)
    l2, Y, g2 = orc.head(S, y, "softmax", lam)
    Sp = np.maximum(S, 0)
    ce = -(Sp[np.arange(n), y] - logsumexp(Sp, axis=1))
    assert abs(l2 - np.sum(lam * ce)) < 1e-13
    np.testing.assert_allclose(g2, lam[:, None] * (Y - np.eye(C)[y]) * (S > 0), atol=1e-16)


def test_permutation_equivariance():
    """Relabelling subgraph nodes permutes P, H, dX and leaves dW unchanged."""
    g = rand_graph(40, 6.0, 26)
    rng = np.random.default_rng(27)
    perm = rng.permutation(g.n)       # new id of old node i is inv[i]
    inv = np.argsort(perm)            # old node perm[k] gets new id k
    Ad = dense_adj(g)
    Ap = Ad[np.ix_(perm, perm)]
    ip = np.concatenate([[0], np.cumsum(Ap.sum(1))]).astype(np.int64)
    ix = np.concatenate([np.nonzero(r)[0] for r in Ap]).astype(np.int32)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    B = orc.normalize(ip, ix, orc.NORM_ROW_SELF)
    X = rng.standard_normal((g.n, 5)); W = rng.standard_normal((5, 3)); dH = rng.standard_normal((g.n, 3))
    P, Z, H = orc.layer_forward(A, X, W)
    Pb, Zb, Hb = orc.layer_forward(B, X[perm], W)
    np.testing.assert_allclose(Hb, H[perm], atol=1e-13)
    _, dW, _, dX = orc.layer_backward(A, P, Z, dH, W)
    _, dWb, _, dXb = orc.layer_backward(B, Pb, Zb, dH[perm], W)
    np.testing.assert_allclose(dWb, dW, atol=1e-12)
    np.testing.assert_allclose(dXb, dX[perm], atol=1e-13)
    assert inv[perm[3]] == 3
