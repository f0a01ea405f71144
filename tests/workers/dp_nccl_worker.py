"""torchrun worker of tests/test_gpu_dp_multi.py (one process per GPU, >= 2 GPUs): the
data-parallel step of SURVEY §8(e) through the C ABI -- each rank runs GCNStep on a subgraph
and gsg_allreduce_grads (NCCL ncclAvg, on gsg's own communicator) averages the flat gradient
buffer -- checked two ways:
  (a) the same subgraph on every rank: mean(dW) equals the rank's own single-GPU dW (1e-6);
  (b) a distinct seeded subgraph per rank: mean(dW) equals the mean of every rank's fp64
      oracle dW (max-normalized error <= 5e-3: TF32 GEMMs).
Rank 0 writes a JSON verdict to argv[1]."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as orc  # noqa: E402
import paper_2010_03166_b200 as gsg  # noqa: E402
import workload as wl  # noqa: E402
from paper_2010_03166_b200 import dp  # noqa: E402
from paper_2010_03166_b200.step import GCNStep  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def run_step(ctx, cfg, g, inp, comm):
    sg = ctx.upload(g.indptr, g.indices, validate=True)
    step = GCNStep(ctx, cfg.dims, g.n, cfg.head, cfg.classes, cfg.precision, device=ctx.device,
                   weights=inp.Ws, w_mlp=inp.W_mlp)
    X = torch.zeros((g.n, wl.ld_for(cfg.dims[0])), device=ctx.device)[:, :cfg.dims[0]]
    X.copy_(torch.from_numpy(inp.X))
    labels = torch.from_numpy(inp.labels).to(ctx.device)
    step.forward_backward(sg, X, labels=labels, comm=comm)
    if comm is not None:
        ctx.nccl_wait(comm, 120000)
    ctx.sync()
    grads = [w.cpu().numpy().astype(np.float64) for w in step.dW] + [step.dWm.cpu().numpy().astype(np.float64)]
    sg.free()
    return grads


def main(out_path):
    rank, world, local = (int(os.environ[k]) for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = gsg.Context(local)
    uid = dp.broadcast_bytes(ctx.nccl_unique_id() if rank == 0 else None)
    comm = ctx.nccl_comm_init(world, rank, uid)
    cfg = wl.tiny_config(n_parent=4000, mean_deg=12.0, n=640, m=64, dims=(48, 96, 64), head="softmax",
                         classes=10)
    res = {"world": world}
    # (a) identical subgraph and inputs on every rank
    g0 = wl.sample_subgraph(cfg, 0, 0)
    inp0 = wl.make_inputs(cfg, g0.n, 0, 0)
    single = run_step(ctx, cfg, g0, inp0, None)
    meaned = run_step(ctx, cfg, g0, inp0, comm)
    res["identical_rel"] = max(rel(a, b) for a, b in zip(meaned, single))
    # (b) own subgraph per rank
    g = wl.sample_subgraph(cfg, 0, rank)
    inp = wl.make_inputs(cfg, g.n, 0, rank)
    mine = run_step(ctx, cfg, g, inp, comm)
    A = orc.normalize(g.indptr, g.indices, orc.NORM_ROW_SELF)
    o = orc.model_step(A, inp.X, inp.Ws, inp.W_mlp, inp.labels, "softmax")
    ref = dp.mean_grads_reference([torch.from_numpy(x) for x in o["dW"] + [o["dW_mlp"]]],
                                  device=torch.device("cuda", local))
    res["distinct_rel"] = max(rel(a, b.cpu().numpy()) for a, b in zip(mine, ref))
    # the subgraphs really differ across ranks
    nodes = [None] * world
    dist.all_gather_object(nodes, g.nodes.tolist())
    res["distinct_subgraphs"] = len({tuple(x) for x in nodes}) == world
    allres = [None] * world
    dist.all_gather_object(allres, res)
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump(allres, f)
    ctx.nccl_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
