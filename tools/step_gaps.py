"""Measurement tool: kernel timeline of one graph-replayed config-5 step (CUPTI through
torch.profiler): per-kernel start / duration, and the idle gaps between consecutive kernels on
the step's stream -- the upper bound of what launch-latency hiding (e.g. programmatic dependent
launch) could save. CFG selects the config (default 5)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2010_03166_b200 as gsg  # noqa: E402
import workload as wl  # noqa: E402
from paper_2010_03166_b200.step import GCNStep  # noqa: E402


def main():
    cfg = wl.CONFIGS[int(os.environ.get("CFG", "5"))]
    g = wl.sample_subgraph(cfg)
    inp = wl.make_inputs(cfg, g.n)
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    with torch.cuda.stream(stream):
        sg = ctx.upload(g.indptr, g.indices)
        sg.normalize()
        step = GCNStep(ctx, cfg.dims, g.n, cfg.head, cfg.classes, cfg.precision, weights=inp.Ws, w_mlp=inp.W_mlp)
        X = torch.zeros((g.n, wl.ld_for(cfg.dims[0])), device="cuda")[:, :cfg.dims[0]]
        X.copy_(torch.from_numpy(inp.X))
        labels = None if inp.labels is None else torch.from_numpy(inp.labels).cuda()
        dH = None
        if inp.dH is not None:
            dH = torch.zeros((g.n, wl.ld_for(cfg.dims[-1])), device="cuda")[:, :cfg.dims[-1]]
            dH.copy_(torch.from_numpy(inp.dH))
        for _ in range(3):
            step.forward_backward(sg, X, labels=labels, dH_top=dH)
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step.forward_backward(sg, X, labels=labels, dH_top=dH)
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.name and "Memcpy" not in e.name]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    # the last replay: kernels after the largest idle gap before it
    steps, cur = [], [ks[0]]
    for k in ks[1:]:
        if k[0] - cur[-1][1] > 200:      # > 200 us idle: next replay
            steps.append(cur)
            cur = [k]
        else:
            cur.append(k)
    steps.append(cur)
    last = steps[-1]
    t0 = last[0][0]
    span = max(k[1] for k in last) - t0
    busy, gaps, end = 0.0, [], t0
    for s, e, n in last:
        if s > end:
            gaps.append((round(s - end, 2), n[:50]))
        busy += max(0.0, e - max(s, end))
        end = max(end, e)
    print(json.dumps({"config": cfg.cid, "kernels": len(last), "span_us": round(span, 1),
                      "busy_us": round(busy, 1), "idle_us": round(span - busy, 1),
                      "gaps_us": sorted(gaps, reverse=True)[:12]}, indent=1))
    import re

    def short(n):  # the kernel's own name out of the (static-prefixed) mangled symbol: <len>k_name
        m = re.search(r"::(k_[A-Za-z0-9_]+)\s*[<(]", n)  # demangled
        if m:
            return m.group(1)
        for m in re.finditer(r"(\d+)(k_[A-Za-z0-9_]+)", n):
            digits, ident = m.group(1), m.group(2)
            for i in range(len(digits)):  # the length prefix may follow other digits (a hash)
                ln = int(digits[i:])
                if 2 <= ln <= len(ident) and (ln == len(ident) or not ident[ln].islower()):
                    return ident[:ln]
        return n[:60]

    per = {}
    for s, e, n in last:
        print(f"{s - t0:9.1f} {e - s:8.1f}  {short(n):24s} {n[:90]}")
        k = short(n)
        per[k] = per.get(k, 0.0) + (e - s)
    print(json.dumps({"kernel_us_in_span": {k: round(v, 1) for k, v in sorted(per.items(), key=lambda x: -x[1])}}, indent=1))


if __name__ == "__main__":
    main()
