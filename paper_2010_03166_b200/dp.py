"""Data-parallel plumbing of the step ("sampling and GNN
computation ... without any dependency constraints"): every rank trains on its own seeded
subgraphs with replicated weights; the only exchange is the mean of the weight gradients
(gsg_allreduce_grads over NCCL on GPUs). Timing is the max over ranks, work the sum.

These helpers are backend-agnostic torch.distributed calls so that the host-side logic is
exercised by world-size-2 gloo tests on the CPU (tests/test_dp_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def reduce_timing(ms: float, work: float, device=None):
    """Return (max over ranks of the timed region in ms, sum over ranks of the work)."""
    t = torch.tensor([ms, work], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        m = t[:1].clone()
        w = t[1:].clone()
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        dist.all_reduce(w, op=dist.ReduceOp.SUM)
        return float(m.item()), float(w.item())
    return float(t[0].item()), float(t[1].item())


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) from `src` to every rank."""
    obj = [payload]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(obj, src=src)
    return obj[0]


def mean_grads_reference(grads: list, device=None) -> list:
    """torch.distributed mean of each gradient tensor (cross-check for gsg_allreduce_grads)."""
    out = []
    world = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
    for g in grads:
        t = torch.as_tensor(g, device=device).clone()
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= world
        out.append(t)
    return out
