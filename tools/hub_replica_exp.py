"""Experiment (measurement only): do L2-slice hot spots from heavily referenced X rows limit the
SpMM? The references to the K most referenced columns are spread round-robin over R replica rows
(extra isolated nodes appended to the graph, X rows copied), so the same gather volume hits R x
more distinct addresses. Same nnz, same row lengths, same f; compares graph-replayed SpMM time.
Env: K (default 256), R list (default 1,2,4,8), F (default 1024)."""
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


def replicate(indptr, indices, n, K, R):
    cnt = np.bincount(indices, minlength=n)
    hot = np.argsort(-cnt)[:K]
    rep = np.full(n, -1, np.int64)
    rep[hot] = np.arange(K)
    ix = indices.astype(np.int64).copy()
    sel = rep[ix] >= 0
    # k-th reference to hot column h -> replica (k mod R); replica 0 is h itself
    order = np.cumsum(sel) - 1
    r = order % R
    tgt = np.where(r == 0, ix, n + rep[ix] * (R - 1) + (r - 1))
    ix = np.where(sel, tgt, ix)
    n2 = n + K * (R - 1)
    out_ix = []
    for i in range(n):
        out_ix.append(np.sort(ix[indptr[i]:indptr[i + 1]]))
    ip2 = np.concatenate([indptr, np.full(n2 - n, indptr[-1], np.int64)])
    return ip2, np.concatenate(out_ix).astype(np.int32), n2, hot, cnt


def main():
    K = int(os.environ.get("K", "256"))
    Rs = [int(x) for x in os.environ.get("R", "1,2,4,8").split(",")]
    f = int(os.environ.get("F", "1024"))
    cfg = wl.CONFIGS[int(os.environ.get("CFG", "5"))]
    g = wl.sample_subgraph(cfg, 0, 0)
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    for R in Rs:
        ip, ix, n2, hot, cnt = replicate(g.indptr, g.indices, g.n, K, R)
        with torch.cuda.stream(stream):
            sg = ctx.upload(ip, ix, validate=False)
            sg.normalize()
            X = torch.randn((n2, f), device="cuda")
            if R > 1:
                X[g.n:] = X[torch.from_numpy(np.repeat(hot, R - 1)).cuda()]
            Y = torch.zeros((n2, f), device="cuda")
        torch.cuda.synchronize()
        ms = timeit(lambda: ctx.spmm(sg, X, Y), iters=20, stream=stream)
        nh = g.nnz + n2
        print(json.dumps({"K": K, "R": R, "f": f, "n": n2, "nnz_hat": nh,
                          "hot_ref_share": float(cnt[hot].sum() / g.nnz), "us": round(ms * 1e3, 2),
                          "gbs": round(4.0 * nh * f / (ms * 1e-3) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
