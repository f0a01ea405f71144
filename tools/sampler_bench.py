"""Measurement tool (NEXT #3): GPU frontier sampling + induction throughput vs the host C++
generator, config 5 shapes (20,000-node frontier subgraphs, m = 3000, 1.6M-node parent).
One JSON line."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_03166_b200 as gsg  # noqa: E402
import workload as wl  # noqa: E402


def main():
    cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    cfg = wl.CONFIGS[cid]
    par = wl.parent_for(cfg)
    p = par.csr()
    out = {"config": cid, "n": cfg.n, "m": cfg.m, "parent_n": p.n, "parent_nnz": p.nnz}
    t0 = time.perf_counter()
    for k in range(3):
        par.frontier_sample(cfg.n, cfg.m, cfg.seed(10, k))
    out["host_cpp_subgraphs_per_s"] = 3 / (time.perf_counter() - t0)
    ctx = gsg.Context(0)
    pg = gsg.ParentGraph(ctx, p.indptr, p.indices)
    pg.sample(cfg.n, cfg.m, 1, count=2).free()  # warm-up
    for count in (1, 16, 148, 444, 888, 1776):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = pg.sample(cfg.n, cfg.m, 1000, count=count)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[f"gpu_batch{count}_s"] = dt
        out[f"gpu_batch{count}_subgraphs_per_s"] = count / dt
        b.free()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
