"""Measurement tool: SpMM effective gather GB/s on random graphs where every row has about the
same degree d (n = 20,000, f = 1024 by default, graph-replayed), so the light-row path
(deg' < 256: one warp per (row, chunk)) and the heavy-row path (deg' >= 256: a CTA per
(row, chunk), 8 warps + smem reduction) are measured separately against the same gather
ceiling (gsg_diag_gather_ceiling on the same X). One JSON line per degree."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2010_03166_b200 as gsg  # noqa: E402
import workload as wl  # noqa: E402
from gemm_bench import timeit  # noqa: E402


def regular_graph(n, d, seed):
    """Symmetric graph with every degree close to d (a union of d/2 random perfect matchings-ish)."""
    rng = np.random.default_rng(seed)
    a = np.repeat(np.arange(n), d // 2)
    b = rng.permutation(a)
    keep = a != b
    a, b = a[keep], b[keep]
    e = np.unique(np.concatenate([a.astype(np.int64) * n + b, b.astype(np.int64) * n + a]))
    r, c = e // n, e % n
    indptr = np.zeros(n + 1, np.int64)
    np.add.at(indptr, r + 1, 1)
    return wl.CSR(np.cumsum(indptr), c.astype(np.int32))


def main():
    n = int(os.environ.get("N", "20000"))
    f = int(os.environ.get("F", "1024"))
    degs = [int(x) for x in os.environ.get("DEGS", "32,64,128,200,250,260,300,450,600,1200").split(",")]
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    X = torch.randn((n, wl.ld_for(f)), device="cuda")[:, :f]
    Y = torch.zeros((n, wl.ld_for(f)), device="cuda")[:, :f]
    ceil = ctx.diag_gather_ceiling(X, min(256, f))
    for d in degs:
        g = regular_graph(n, d, d)
        with torch.cuda.stream(stream):
            sg = ctx.upload(g.indptr, g.indices, validate=False).normalize()
        torch.cuda.synchronize()
        nh = g.nnz + n
        with torch.cuda.stream(stream):
            ms = timeit(lambda: ctx.spmm(sg, X, Y), iters=20, stream=stream)
        eff = 4.0 * nh * f + 8.0 * nh + 4.0 * (n + 1) + 4.0 * n * f
        deg = np.diff(g.indptr) + 1
        print(json.dumps({"deg_target": d, "deg_mean": float(deg.mean()), "heavy_rows_frac": float((deg >= 256).mean()),
                          "us": round(ms * 1e3, 1), "gbs": round(eff / (ms * 1e-3) / 1e9, 1),
                          "ceiling_gbs": round(ceil, 1), "frac": round(eff / (ms * 1e-3) / 1e9 / ceil, 3)}), flush=True)
        sg.free()


if __name__ == "__main__":
    main()
