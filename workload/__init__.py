"""Seeded synthetic workload generator shared by the oracle and the CUDA path.

SURVEY §8(a) row a0 (SUPPORT) and §8(d) "Concrete synthetic inputs". This module holds
none of the GCN layer's arithmetic: it emits integer CSR structure (via the C++ library
``libgsgen.so``) and seeded random dense inputs (numpy PCG64). Both ``oracle/`` and
``paper_2010_03166_b200/`` consume these arrays as *inputs*; neither imports the other.

Stand-ins: the paper's PPI / Reddit / Yelp / Amazon datasets (Table 1)
are not available; each config reproduces node count, mean degree, attribute width and
class count with a Chung-Lu power-law parent and a frontier-sampled subgraph (Alg. 2,
PAPER.md:366-385).
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgsgen.so")
_lib = None

S0 = 20103166  # base seed (SURVEY §8(d) "Seeds")


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        L.gsgen_parent_build.restype = vp
        L.gsgen_parent_build.argtypes = [i64, dbl, dbl, dbl, u64]
        L.gsgen_graph_free.argtypes = [vp]
        L.gsgen_graph_n.restype = i64
        L.gsgen_graph_n.argtypes = [vp]
        L.gsgen_graph_nnz.restype = i64
        L.gsgen_graph_nnz.argtypes = [vp]
        L.gsgen_graph_copy.argtypes = [vp, vp, vp]
        L.gsgen_graph_from_csr.restype = vp
        L.gsgen_graph_from_csr.argtypes = [i64, vp, vp]
        L.gsgen_frontier_sample.restype = vp
        L.gsgen_frontier_sample.argtypes = [vp, i64, i64, i64, u64]
        L.gsgen_subgraph_free.argtypes = [vp]
        L.gsgen_subgraph_n.restype = i64
        L.gsgen_subgraph_n.argtypes = [vp]
        L.gsgen_subgraph_nnz.restype = i64
        L.gsgen_subgraph_nnz.argtypes = [vp]
        L.gsgen_subgraph_copy.argtypes = [vp, vp, vp, vp]
        L.gsgen_induce.restype = vp
        L.gsgen_induce.argtypes = [vp, i64, vp]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class CSR:
    """Symmetric CSR without self loops: int64 indptr[n+1], int32 indices[nnz] (ascending rows)."""
    indptr: np.ndarray
    indices: np.ndarray
    nodes: np.ndarray | None = None  # parent ids (ascending) for a sampled subgraph

    @property
    def n(self) -> int:
        return int(self.indptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def stats(self) -> dict:
        d = self.degrees()
        if d.size == 0:
            return {"n": 0, "nnz": 0}
        return {"n": self.n, "nnz": self.nnz, "nnz_with_self": self.nnz + self.n,
                "mean_deg": float(d.mean()), "p50_deg": float(np.percentile(d, 50)),
                "p99_deg": float(np.percentile(d, 99)), "max_deg": int(d.max()),
                "frac_deg_le_32": float((d <= 32).mean()), "rows_deg_gt_1024": int((d > 1024).sum())}


class Parent:
    """Chung-Lu power-law parent graph handle (C++ owned)."""

    def __init__(self, n: int, mean_deg: float, gamma: float = 2.1, w_max: float = 0.0, seed: int = 1):
        self._h = lib().gsgen_parent_build(n, float(mean_deg), float(gamma), float(w_max), seed)
        if not self._h:
            raise ValueError("gsgen_parent_build failed (bad parameters)")
        self.n = n

    @classmethod
    def from_csr(cls, csr: CSR) -> "Parent":
        obj = cls.__new__(cls)
        ip = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(csr.indices, dtype=np.int32)
        obj._h = lib().gsgen_graph_from_csr(csr.n, _ptr(ip), _ptr(ix))
        obj.n = csr.n
        return obj

    def csr(self) -> CSR:
        L = lib()
        n, nnz = L.gsgen_graph_n(self._h), L.gsgen_graph_nnz(self._h)
        ip = np.empty(n + 1, np.int64)
        ix = np.empty(nnz, np.int32)
        L.gsgen_graph_copy(self._h, _ptr(ip), _ptr(ix))
        return CSR(ip, ix)

    def frontier_sample(self, n: int, m: int, seed: int, clip: int = 16) -> CSR:
        L = lib()
        h = L.gsgen_frontier_sample(self._h, n, m, clip, seed)
        if not h:
            raise ValueError("frontier sampling failed (m or n too large for the parent)")
        try:
            return _sub_to_csr(h)
        finally:
            L.gsgen_subgraph_free(h)

    def induce(self, nodes: np.ndarray) -> CSR:
        nodes = np.ascontiguousarray(nodes, dtype=np.int64)
        if nodes.size > 1 and not np.all(np.diff(nodes) > 0):
            raise ValueError("nodes must be strictly ascending")
        h = lib().gsgen_induce(self._h, nodes.size, _ptr(nodes))
        try:
            return _sub_to_csr(h)
        finally:
            lib().gsgen_subgraph_free(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.gsgen_graph_free(h)
            self._h = None


def _sub_to_csr(h) -> CSR:
    L = lib()
    n, nnz = L.gsgen_subgraph_n(h), L.gsgen_subgraph_nnz(h)
    ip = np.empty(n + 1, np.int64)
    ix = np.empty(nnz, np.int32)
    nodes = np.empty(n, np.int64)
    L.gsgen_subgraph_copy(h, _ptr(ip), _ptr(ix), _ptr(nodes))
    return CSR(ip, ix, nodes)


# ------------------------------------------------------------------------------------------
# Configs (BASELINE.json "configs", knobs per SURVEY §8(d) / Appendix A)
# ------------------------------------------------------------------------------------------
@dataclass
class Config:
    cid: int
    name: str
    parent_n: int
    parent_mean_deg: float
    gamma: float
    w_max: float          # 0 => structural cutoff sqrt(n * mean_deg)
    n: int                # subgraph node budget
    m: int                # frontier size
    dims: list            # [f0, f1, ..., fL]
    precision: str        # "tf32" | "bf16" | "fp32x3" (3xTF32: fp32-accurate GEMMs, configs 1-2 "fp32")
    head: str             # "none" | "softmax" | "sigmoid"
    classes: int = 0
    label_p: float = 0.05
    dp: bool = False
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def L(self) -> int:
        return len(self.dims) - 1

    def seed(self, tag: int, k: int = 0, r: int = 0) -> int:
        """Seed for an input stream: tag 1 parent, 2 X, 3 dH/labels, 10 sampler, 20+l weight l.

        Per-subgraph streams (sampler, X, dH/labels) add 1000*k (pool index) + 10**6*r (rank);
        weights are replicated across ranks (data parallelism)."""
        return S0 + 100 * self.cid + tag + 1000 * k + 1_000_000 * r


CONFIGS = {
    1: Config(1, "ppi-like", 20_000, 15.0, 2.1, 0.0, 2_000, 200, [50, 128], "fp32x3", "none"),
    2: Config(2, "reddit-like", 230_000, 50.0, 2.1, 1250.0, 8_000, 1000, [602, 512, 512], "fp32x3", "softmax", 41),
    3: Config(3, "yelp-like", 720_000, 10.0, 2.1, 0.0, 12_000, 1000, [300, 512, 512, 512], "tf32", "sigmoid", 100),
    4: Config(4, "amazon-deep", 1_600_000, 4.5, 2.1, 2.5e5, 16_000, 1000, [200, 1024, 1024, 1024, 1024, 1024], "bf16", "none"),
    5: Config(5, "amazon-dp", 1_600_000, 80.0, 2.1, 0.0, 20_000, 3000, [200, 1024, 1024, 1024], "tf32", "sigmoid", 107, dp=True),
}


def tiny_config(n_parent=400, mean_deg=8.0, n=64, m=16, dims=(12, 16), head="none", classes=0,
                precision="tf32", cid=90) -> Config:
    """Small configs for parity tests the oracle finishes in well under a second."""
    return Config(cid, f"tiny{cid}", n_parent, mean_deg, 2.1, 0.0, n, m, list(dims), precision, head, classes)


def ld_for(f: int, align: int = 8) -> int:
    """Row stride (elements) for a width-f row-major buffer: 32-byte (sector) aligned fp32 rows,
    which also satisfies the 16-byte TMA stride rule (gsg.h "Layout")."""
    return int(math.ceil(f / align) * align)


_PARENT_CACHE: dict = {}


def parent_for(cfg: Config) -> Parent:
    key = (cfg.parent_n, cfg.parent_mean_deg, cfg.gamma, cfg.w_max, cfg.seed(1))
    p = _PARENT_CACHE.get(key)
    if p is None:
        p = Parent(cfg.parent_n, cfg.parent_mean_deg, cfg.gamma, cfg.w_max, cfg.seed(1))
        _PARENT_CACHE[key] = p
    return p


def sample_subgraph(cfg: Config, k: int = 0, r: int = 0) -> CSR:
    return parent_for(cfg).frontier_sample(cfg.n, cfg.m, cfg.seed(10, k, r))


def block_diag(parts: list) -> CSR:
    """Disjoint union of subgraphs as one CSR (block-diagonal adjacency; node ids of part b are
    offset by the sizes of parts 0..b-1). The paper trains on independent subgraphs with no
    dependency between them; batching B of them per launch with a shared W is the
    same computation as B separate layers, so a small config can fill the GPU (SURVEY §8(d),
    config 1 "batched variant"). Pure structure: no method arithmetic."""
    n_off, e_off = 0, 0
    ips, ixs = [np.zeros(1, np.int64)], []
    for c in parts:
        ips.append(c.indptr[1:].astype(np.int64) + e_off)
        ixs.append(c.indices.astype(np.int64) + n_off)
        n_off += c.n
        e_off += c.nnz
    ix = np.concatenate(ixs) if ixs else np.zeros(0, np.int64)
    if n_off >= 2**31:
        raise ValueError("batched subgraph exceeds int32 node ids")
    return CSR(np.concatenate(ips), ix.astype(np.int32))


def sample_batch(cfg: Config, batch: int, slot: int = 0, r: int = 0) -> CSR:
    """B independent subgraphs (pool indices slot*B .. slot*B+B-1) as one block-diagonal CSR."""
    return block_diag([sample_subgraph(cfg, slot * batch + b, r) for b in range(batch)])


@dataclass
class Inputs:
    """Dense seeded inputs for one subgraph (unpadded, row-major float32)."""
    X: np.ndarray                      # [n, f0] ~ N(0,1)
    Ws: list                           # [f_{l-1}, f_l] Glorot-uniform, l = 1..L
    W_mlp: np.ndarray | None           # [f_L, C]
    dH: np.ndarray | None              # [n, f_L] ~ N(0,1) (configs without a head)
    labels: np.ndarray | None          # softmax: int32 [n]; sigmoid: uint8 [n, C]


def glorot(rng: np.random.Generator, fi: int, fo: int) -> np.ndarray:
    a = math.sqrt(6.0 / (fi + fo))
    return rng.uniform(-a, a, size=(fi, fo)).astype(np.float32)


def make_inputs(cfg: Config, n: int, k: int = 0, r: int = 0) -> Inputs:
    rx = np.random.default_rng(cfg.seed(2, k, r))
    X = rx.standard_normal((n, cfg.dims[0]), dtype=np.float32)
    Ws = [glorot(np.random.default_rng(cfg.seed(20 + l)), cfg.dims[l - 1], cfg.dims[l])
          for l in range(1, cfg.L + 1)]
    W_mlp = dH = labels = None
    ry = np.random.default_rng(cfg.seed(3, k, r))
    if cfg.head == "none":
        dH = ry.standard_normal((n, cfg.dims[-1]), dtype=np.float32)
    else:
        W_mlp = glorot(np.random.default_rng(cfg.seed(20 + cfg.L + 1)), cfg.dims[-1], cfg.classes)
        if cfg.head == "softmax":
            labels = ry.integers(0, cfg.classes, size=n, dtype=np.int32)
        else:
            labels = (ry.random((n, cfg.classes)) < cfg.label_p).astype(np.uint8)
    return Inputs(X, Ws, W_mlp, dH, labels)


def random_values(csr: CSR, seed: int) -> np.ndarray:
    """Positive random edge weights (general weighted Â input, e.g. GraphSAINT-style)."""
    return np.random.default_rng(seed).uniform(0.1, 1.0, size=csr.nnz).astype(np.float32)


def config_table() -> str:
    return json.dumps({c: vars(v) for c, v in CONFIGS.items()}, indent=1, default=str)
