"""Measurement tool: the SpMM (a2 / a7) alone on a config's subgraph at the widths the step
runs (config 5: f = 1024 and 200), graph-replayed, effective gather GB/s.
LD_ALIGN (elements, default 8) sets the row stride alignment of X and Y. One JSON line per
width."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2010_03166_b200 as gsg  # noqa: E402
import workload as wl  # noqa: E402
from gemm_bench import timeit  # noqa: E402


def main():
    cfgid = int(os.environ.get("CFG", "5"))
    widths = [int(x) for x in os.environ.get("WIDTHS", "1024,200").split(",")]
    cfg = wl.CONFIGS[cfgid]
    g = wl.sample_subgraph(cfg, 0, 0)
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    with torch.cuda.stream(stream):
        sg = ctx.upload(g.indptr, g.indices, validate=False)
        sg.normalize()
    torch.cuda.synchronize()
    nh = g.nnz + g.n
    for f in widths:
        ld = wl.ld_for(f, int(os.environ.get("LD_ALIGN", "8")))
        X = torch.randn((g.n, ld), device="cuda")[:, :f]
        Y = torch.zeros((g.n, ld), device="cuda")[:, :f]
        res = {}
        for tr in (0, 1):
            with torch.cuda.stream(stream):
                ms = timeit(lambda: ctx.spmm(sg, X, Y, transpose=bool(tr)), iters=20, stream=stream)
            eff = 4.0 * nh * f + 8.0 * nh + 4.0 * (g.n + 1) + 4.0 * g.n * f
            res["T" if tr else "N"] = {"us": round(ms * 1e3, 2), "gbs": round(eff / (ms * 1e-3) / 1e9, 1)}
        print(json.dumps({"cfg": cfgid, "f": f, "n": g.n, "nnz_hat": nh, "ld": ld, **res}), flush=True)


if __name__ == "__main__":
    main()
