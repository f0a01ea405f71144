"""fp64 CPU oracle for the GCN-layer hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. It shares no code
with ``paper_2010_03166_b200`` (the CUDA path) and never imports it.

The arithmetic lives in ``oracle.c`` (plain loops, double precision); this wrapper only
marshals numpy arrays (upcasting inputs to float64) and composes the per-layer steps in
the paper's order:

  forward  (Eq. 5):  P = Â X ; Z = P W ; H = ReLU(Z)
  backward (with Eq. 13 at P:704): dZ = dH ⊙ 1[Z > 0] ; dW = Pᵀ dZ ;
                                          T = dZ Wᵀ ; dX = Âᵀ T
  head     (Eqs. 2-4 / 9-11)

Parity status: every function below is pinned by tests/test_oracle_pins.py (closed forms,
dense brute force, the adjoint identity, central finite differences, the SPEC examples);
none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

NORM_ROW_SELF, NORM_SYM_SELF, NORM_ROW, NORM_VALUES = 0, 1, 2, 3


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make oracle`")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64, dbl, cint = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.oracle_nnz_hat.restype = i64
        L.oracle_nnz_hat.argtypes = [i32, i64, cint]
        L.oracle_normalize.restype = None
        L.oracle_normalize.argtypes = [i32, vp, vp, vp, cint, vp, vp, vp]
        L.oracle_transpose_alg4.restype = cint
        L.oracle_transpose_alg4.argtypes = [i32, vp, vp, vp, vp]
        L.oracle_spmm.restype = None
        L.oracle_spmm.argtypes = [i32, i32, vp, vp, vp, vp, i64, i32, i32, vp, i64]
        L.oracle_spmm_t_scatter.restype = None
        L.oracle_spmm_t_scatter.argtypes = [i32, i32, vp, vp, vp, vp, i64, i32, i32, vp, i64]
        L.oracle_gemm.restype = None
        L.oracle_gemm.argtypes = [i32, i32, i32, vp, i64, cint, vp, i64, cint, vp, i64]
        L.oracle_frontier_sample.restype = i32
        L.oracle_frontier_sample.argtypes = [i64, vp, vp, i32, i32, i32, ctypes.c_uint64, vp]
        L.oracle_induce.restype = i64
        L.oracle_induce.argtypes = [i64, vp, vp, i32, vp, vp, vp]
        L.oracle_head.restype = dbl
        L.oracle_head.argtypes = [i32, i32, vp, i64, cint, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class AHat:
    """Â in CSR (self loops inserted in the *_SELF modes), fp64 values."""
    indptr: np.ndarray   # int64 [n+1]
    idx: np.ndarray      # int32 [nnz_hat]
    val: np.ndarray      # float64 [nnz_hat]

    @property
    def n(self) -> int:
        return self.indptr.shape[0] - 1

    def dense(self) -> np.ndarray:
        D = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.indptr[i], self.indptr[i + 1]):
                D[i, self.idx[k]] += self.val[k]
        return D


def normalize(indptr, indices, mode: int = NORM_ROW_SELF, values=None) -> AHat:
    """Â per SURVEY §8(c) step 1 (Eq. 5; row mode R1; GraphSAGE P:131; weighted P:668)."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    n, nnz = ip.shape[0] - 1, int(ip[-1])
    if mode == NORM_VALUES and values is None:
        raise ValueError("NORM_VALUES needs values")
    vals = _f64(values) if values is not None else np.zeros(1)
    nh = lib().oracle_nnz_hat(n, nnz, mode)
    ipo = np.empty(n + 1, np.int64)
    ixo = np.empty(max(nh, 1), np.int32)
    vo = np.empty(max(nh, 1), np.float64)
    lib().oracle_normalize(n, _p(ip), _p(ix), _p(vals), mode, _p(ipo), _p(ixo), _p(vo))
    return AHat(ipo, ixo[:nh], vo[:nh])


def transpose_alg4(A: AHat) -> np.ndarray:
    """DataTrans of Alg. 4: values of Âᵀ on Â's (shared) structure."""
    out = np.full(max(A.val.shape[0], 1), np.nan)
    rc = lib().oracle_transpose_alg4(A.n, _p(A.indptr), _p(A.idx), _p(_f64(A.val)), _p(out))
    if rc != 0:
        raise ValueError("Alg. 4 precondition violated (asymmetric structure)")
    return out[: A.val.shape[0]]


def spmm(A: AHat, X, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """P = Â X (rows r0..r1; other rows left zero)."""
    X = _f64(X)
    n, f = X.shape
    r1 = n if r1 is None else r1
    P = np.zeros((n, f))
    lib().oracle_spmm(n, f, _p(A.indptr), _p(A.idx), _p(_f64(A.val)), _p(X), f, r0, r1, _p(P), f)
    return P


def spmm_t(A: AHat, T, r0: int = 0, r1: int | None = None) -> np.ndarray:
    """dX = Âᵀ T by scatter from the definition of the transpose (contributions of rows r0..r1)."""
    T = _f64(T)
    n, f = T.shape
    r1 = n if r1 is None else r1
    dX = np.empty((n, f))
    lib().oracle_spmm_t_scatter(n, f, _p(A.indptr), _p(A.idx), _p(_f64(A.val)), _p(T), f, r0, r1, _p(dX), f)
    return dX


def gemm(A, B, transA: bool = False, transB: bool = False) -> np.ndarray:
    """C = op(A) op(B) by triple loops."""
    A, B = _f64(A), _f64(B)
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    Kb = B.shape[1] if transB else B.shape[0]
    if K != Kb:
        raise ValueError(f"inner dims {K} != {Kb}")
    C = np.empty((M, N))
    lib().oracle_gemm(M, N, K, _p(A), A.shape[1], int(transA), _p(B), B.shape[1], int(transB), _p(C), N)
    return C


def relu(Z):
    return np.maximum(Z, 0.0)


def layer_forward(A: AHat, X, W):
    """GCN layer forward, Eq. 5 under the fixed chain order (ÂX)W: returns P, Z, H."""
    P = spmm(A, X)
    Z = gemm(P, W)
    return P, Z, relu(Z)


def relu_mask(dH, Z):
    """mask(·) = ReLU' gate from the cached pre-activation, ReLU'(0) = 0 (R4)."""
    return np.where(_f64(Z) > 0, _f64(dH), 0.0)


def layer_backward(A: AHat, P, Z, dH, W, need_dX: bool = True, premasked: bool = False):
    """GCN layer backward (P:719 with Eq. 13): dZ, dW = Pᵀ dZ, T = dZ Wᵀ, dX = Âᵀ T."""
    dZ = _f64(dH) if premasked else relu_mask(dH, Z)
    dW = gemm(P, dZ, transA=True)
    T = gemm(dZ, W, transB=True)
    dX = spmm_t(A, T) if need_dX else None
    return dZ, dW, T, dX


def sage_forward(Abar: AHat, X, Ws, Wn):
    """GraphSAGE layer, Eq. 1 with Ã = D⁻¹A (normalize(..., NORM_ROW)); column layout
    [self | neighbor] per the slices of Eqs. 12-15 (reading R21). Returns P = ÃX, Z, H."""
    X = _f64(X)
    P = spmm(Abar, X)
    Z = np.hstack([gemm(X, Ws), gemm(P, Wn)])
    return P, Z, relu(Z)


def sage_backward(Abar: AHat, X, P, Z, dH, Ws, Wn, premasked: bool = False):
    """Eqs. 12-15: dW_s = Xᵀ mask(dH)[:, :f/2], dW_n = (ÃX)ᵀ mask(dH)[:, f/2:],
    dX = mask(dH)[:, :f/2] W_sᵀ + Ãᵀ mask(dH)[:, f/2:] W_nᵀ."""
    dZ = _f64(dH) if premasked else relu_mask(dH, Z)
    fh = np.asarray(Ws).shape[1]
    dZs, dZn = np.ascontiguousarray(dZ[:, :fh]), np.ascontiguousarray(dZ[:, fh:])
    dWs = gemm(X, dZs, transA=True)
    dWn = gemm(P, dZn, transA=True)
    dX = gemm(dZs, Ws, transB=True) + spmm_t(Abar, gemm(dZn, Wn, transB=True))
    return dZ, dWs, dWn, dX


def frontier_sample(indptr, indices, n: int, m: int, clip: int, seed: int) -> np.ndarray:
    """Alg. 2 (reading R9) with the counter-based draws of include/gsg.h; returns the
    ascending node list V_s (parent ids)."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    out = np.empty(n, np.int32)
    nv = lib().oracle_frontier_sample(ip.shape[0] - 1, _p(ip), _p(ix), n, m, clip, seed, _p(out))
    return out[:nv]


def induce(indptr, indices, nodes):
    """Induced subgraph on an ascending node list (Alg. 2 line 9): (indptr int64, indices int32)."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    nd = np.ascontiguousarray(nodes, dtype=np.int32)
    sp = np.empty(nd.shape[0] + 1, np.int64)
    nnz = lib().oracle_induce(ip.shape[0] - 1, _p(ip), _p(ix), nd.shape[0], _p(nd), _p(sp), None)
    si = np.empty(max(nnz, 1), np.int32)
    lib().oracle_induce(ip.shape[0] - 1, _p(ip), _p(ix), nd.shape[0], _p(nd), _p(sp), _p(si))
    return sp, si[:nnz]


def head(S, labels, kind: str, node_w=None):
    """Eqs. 2-4 forward + Eqs. 9-10 backward. Returns loss, Y, dS."""
    S = _f64(S)
    n, C = S.shape
    Y = np.empty((n, C))
    dS = np.empty((n, C))
    if kind == "softmax":
        cls = np.ascontiguousarray(labels, dtype=np.int32)
        ind = np.zeros(1, np.uint8)
        k = 0
    elif kind == "sigmoid":
        ind = np.ascontiguousarray(labels, dtype=np.uint8)
        cls = np.zeros(1, np.int32)
        k = 1
    else:
        raise ValueError(kind)
    w = None if node_w is None else _f64(node_w)
    loss = lib().oracle_head(n, C, _p(S), C, k, _p(cls), _p(ind), None if w is None else _p(w), _p(Y), _p(dS))
    return loss, Y, dS


def head_backward(H_L, dS, W_mlp):
    """dW_mlp = H_Lᵀ dS ; dH_L = dS W_mlpᵀ (Eq. 10-11)."""
    return gemm(H_L, dS, transA=True), gemm(dS, W_mlp, transB=True)


def model_step(A: AHat, X, Ws, W_mlp=None, labels=None, head_kind="none", dH_top=None):
    """Full L-layer forward + backward (Alg. 1 lines 7-13) with the fixed chain
    order; returns a dict of every intermediate (fp64)."""
    out = {"P": [], "Z": [], "H": [], "dZ": [], "dW": [], "T": [], "dX": []}
    h = _f64(X)
    for W in Ws:
        P, Z, H = layer_forward(A, h, W)
        out["P"].append(P); out["Z"].append(Z); out["H"].append(H)
        h = H
    if head_kind == "none":
        dH = _f64(dH_top)
        out["loss"] = None
    else:
        S = gemm(h, W_mlp)
        loss, Y, dS = head(S, labels, head_kind)
        dWm, dH = head_backward(h, dS, W_mlp)
        out.update(S=S, loss=loss, Y=Y, dS=dS, dW_mlp=dWm, dH_top=dH)
    for l in range(len(Ws) - 1, -1, -1):
        dZ, dW, T, dX = layer_backward(A, out["P"][l], out["Z"][l], dH, Ws[l])
        out["dZ"].insert(0, dZ); out["dW"].insert(0, dW); out["T"].insert(0, T); out["dX"].insert(0, dX)
        dH = dX
    return out
