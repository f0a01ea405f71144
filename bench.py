#!/usr/bin/env python
"""Benchmark of the GCN-layer hot path (BASELINE.json metric: "GCN layer fwd+bwd: subgraph
edge·features/s and % HBM/tensor roofline") on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

A "step" is one pass of every SURVEY §8(a) row over one sampled subgraph per GPU: normalize
(a1), the L layers' forward (a2, a3), the classifier head (a8), the L layers' backward
(a4-a7) and, for N > 1, the NCCL mean of all dW (a9). Default workload: config 5 (the
data-parallel config BASELINE.json quotes at 1/2/4/8 GPUs): 20,000-node frontier subgraphs
of a 1.6M-node power-law parent, GCN 200->1024->1024->1024, 107-way sigmoid head, TF32
GEMMs, fp32 SpMM. Each rank takes its own seeded subgraphs (weak scaling); a pool of
--pool pre-sampled subgraphs per rank rotates across steps (Alg. 7's pool).

value  = (sum over ranks of 2*nnz'*f_in edge-features per layer, all layers, all timed steps)
         / (max over ranks of the device-timed region) -- inputs resident in HBM.
e2e    = the same work measured through the same C-ABI calls with the step's inputs copied
         from pinned host memory (CSR + X + labels) and the loss read back every step.
Launch for N > 1: torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL logs at INFO (communicator init: ranks, NVLink/NVLS topology, tuning tables) into a
# per-process file, which bench.py copies to stderr after the first all-reduce and parses for
# the JSON line (ranks seen, NVLS); stdout carries exactly the one JSON line the driver reads.
# (the image exports NCCL_DEBUG=VERSION, so the level is set explicitly; GSG_NCCL_DEBUG overrides)
os.environ["NCCL_DEBUG"] = os.environ.get("GSG_NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV,TUNING,NVLS")
if "NCCL_DEBUG_FILE" not in os.environ:
    import tempfile
    os.environ["NCCL_DEBUG_FILE"] = os.path.join(tempfile.gettempdir(), f"gsg_bench_nccl.{os.getpid()}.log")


def nccl_log_summary(echo: bool = True):
    """Copy this process's NCCL debug log to stderr and summarize it: the communicator sizes
    NCCL reported (nRanks), whether NVLS (NVLink SHARP in-switch reduction) was set up, and the
    algorithm lines of the tuning output."""
    import re
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    if not path or "%" in path or not os.path.exists(path):
        return {"log": None}
    with open(path, errors="replace") as f:
        lines = f.read().splitlines()
    if echo:
        for ln in lines:
            print(ln, file=sys.stderr)
        sys.stderr.flush()
    nranks = sorted({int(m.group(1)) for ln in lines for m in [re.search(r"nRanks (\d+)", ln)] if m})
    nvls = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if "NVLS" in ln]
    algo = [ln.split("NCCL INFO", 1)[-1].strip() for ln in lines if re.search(r"Algorithm|AllReduce \|", ln)]
    ver = next((ln.split("NCCL version", 1)[-1].strip() for ln in lines if "NCCL version" in ln), None)
    return {"log": path, "lines": len(lines), "version": ver, "nranks_seen": nranks,
            "nvls_lines": nvls[:6], "nvls": any(("NVLS" in x and "enable" in x.lower()) or "multicast" in x.lower()
                                                  for x in nvls),
            "tuning_lines": algo[:8]}


class stdout_to_stderr:
    """Route file descriptor 1 to stderr for the duration (library banners, e.g. NCCL's)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False

import workload as wl  # noqa: E402

METRIC = "GCN layer fwd+bwd: subgraph edge·features/s and % HBM/tensor roofline"
UNIT = "edge·features/s"


# ------------------------------------------------------------------------------ helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "bf16_tflops": d.get("bf16_tflops", 1590.0),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", 1400.0), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int, period_s: float = 0.02):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period, self._stop = period_s, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[device])
                except ValueError:
                    pass
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ------------------------------------------------------------------------------ oracle leg
class OracleSample:
    """Times the fp64 oracle (oracle/, as it stands) on a bounded row sample of one step of
    this workload: for every layer the aggregation, transform, ReLU' gate, dW, T and the
    scatter-form transpose restricted to output/source rows [0, R) (plus the head on the same
    rows). Stand-in layer inputs are random (values do not affect the oracle's run time)."""

    def __init__(self, cfg, csr, inputs, seed: int = 0):
        import oracle as orc
        self.orc, self.cfg, self.csr, self.inputs = orc, cfg, csr, inputs
        self.A = orc.normalize(csr.indptr, csr.indices, orc.NORM_ROW_SELF)
        rng = np.random.default_rng(seed)
        dims = cfg.dims
        self.hs = [np.ascontiguousarray(inputs.X, np.float64)] + \
            [np.abs(rng.standard_normal((csr.n, f))) for f in dims[1:-1]]
        self.Ws = [np.asarray(w, np.float64) for w in inputs.Ws]
        self.dHs = [rng.standard_normal((csr.n, f)) for f in dims[1:]]
        self.rows = None

    def run(self, R: int):
        orc, cfg, dims, A = self.orc, self.cfg, self.cfg.dims, self.A
        work = 0
        t0 = time.perf_counter()
        for l in range(cfg.L):
            P = orc.spmm(A, self.hs[l], 0, R)
            Z = orc.gemm(P[:R], self.Ws[l])
            dZ = orc.relu_mask(self.dHs[l][:R], Z)
            orc.gemm(P[:R], dZ, transA=True)
            T = np.zeros((self.csr.n, dims[l]))
            T[:R] = orc.gemm(dZ, self.Ws[l], transB=True)
            orc.spmm_t(A, T, 0, R)
            work += 2 * int(A.indptr[R]) * dims[l]
        if cfg.head != "none":
            S = orc.gemm(np.maximum(Z, 0), self.inputs.W_mlp)
            _, _, dS = orc.head(S, self.inputs.labels[:R], cfg.head)
            orc.head_backward(np.maximum(Z, 0), dS, self.inputs.W_mlp)
        return work, time.perf_counter() - t0

    def calibrate(self, target_s: float):
        R = min(64, self.csr.n)
        work, dt = self.run(R)
        while dt < 0.2 * target_s and R < self.csr.n:
            R = min(self.csr.n, max(R + 1, int(R * min(8.0, 0.8 * target_s / max(dt, 1e-3)))))
            work, dt = self.run(R)
        self.rows = R
        return work, dt

    @staticmethod
    def cores():
        return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))

    @staticmethod
    def cpu_model():
        """The host CPU the oracle ran on (/proc/cpuinfo), as BASELINE.md's plan asks."""
        try:
            with open("/proc/cpuinfo") as f:
                for ln in f:
                    if ln.lower().startswith("model name"):
                        return ln.split(":", 1)[1].strip()
        except OSError:
            pass
        import platform
        return platform.processor() or None


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    g = wl.sample_subgraph(cfg, 0, 0)
    inp = wl.make_inputs(cfg, g.n, 0, 0)
    per_step = max(0.5, min(8.0, 120.0 / max(1, args.steps + args.warmup)))
    vals = []
    osamp = OracleSample(cfg, g, inp)
    osamp.calibrate(per_step)  # size the row sample once
    for i in range(args.warmup + args.steps):
        work, dt = osamp.run(osamp.rows)
        if i >= args.warmup:
            vals.append(work / dt)
    value = float(statistics.median(vals)) if vals else 0.0
    info = {"rows": osamp.rows, "cores": osamp.cores()}
    sample = (f"rows [0,{info['rows']}) of rank 0's config-{cfg.cid} subgraph (n={g.n}, nnz'={g.nnz + g.n}): "
              f"all {cfg.L} layers' aggregation, transform, gate, dW, T, transposed scatter + head, fp64")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"config{cfg.cid}:{cfg.name}", "nodes": g.n, "dims": cfg.dims},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "oracle", "sample": sample,
                            "cpu_model": OracleSample.cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_gpu_sampled(args, cfg, ctx, runner, stream, dev, rank, nnz_hint):
    """Training loop fed by the GPU frontier sampler (NEXT #3, Alg. 2 on the device; Alg. 7's pool
    refill): the parent graph, a seeded parent feature matrix and labels live in HBM;
    one gsg_frontier_sample call draws --sampler-pool subgraphs; ONE CUDA graph of the step --
    gsg_sample_load of sample *d_k into a device-sized subgraph (sizes read on the device,
    *d_k advanced by the graph itself), X_s = X[V_s] and label gathers (Alg. 1 line 5),
    normalize, layers, head (per-node loss weights 1/n_k), backward -- is captured per sampled
    batch and replayed once per sample. The timed region covers the sampling calls, the graph
    captures and every replay. Returns edge-features/s of the loop and the sampler's share."""
    import torch
    import paper_2010_03166_b200 as gsg
    P = max(1, args.sampler_pool)
    pc = wl.parent_for(cfg).csr()
    pg = gsg.ParentGraph(ctx, pc.indptr, pc.indices)
    gen = torch.Generator(device=dev)
    gen.manual_seed(cfg.seed(2, 0, rank) + 7)
    f0 = cfg.dims[0]
    n_pad = runner.n_max
    with torch.cuda.stream(stream):
        Xpar = torch.randn((pc.n, wl.ld_for(f0)), device=dev, generator=gen)[:, :f0]
        if cfg.head == "softmax":
            Lpar = torch.randint(0, cfg.classes, (pc.n, 1), device=dev, generator=gen, dtype=torch.int32)
        elif cfg.head == "sigmoid":
            Lpar = (torch.rand((pc.n, cfg.classes), device=dev, generator=gen) < cfg.label_p).to(torch.uint8)
        else:
            Lpar = None
        Xs = torch.zeros((n_pad, wl.ld_for(f0)), device=dev)[:, :f0]
        Ls = None if Lpar is None else torch.zeros((n_pad, Lpar.shape[1]), dtype=Lpar.dtype, device=dev)
        dH = None
        if cfg.head == "none":
            dH = torch.randn((n_pad, wl.ld_for(cfg.dims[-1])), device=dev, generator=gen)[:, :cfg.dims[-1]]
        d_k = torch.zeros(1, dtype=torch.int32, device=dev)
        nodes = torch.zeros(n_pad, dtype=torch.int32, device=dev)
        node_w = torch.zeros(n_pad, dtype=torch.float32, device=dev)
    sgd = ctx.create_device(n_pad, int(2 * nnz_hint))
    seed0 = cfg.seed(10, 0, rank) + 777
    labels = None if Ls is None else (Ls[:, 0] if cfg.head == "softmax" else Ls)

    def one(batch):
        batch.load(ctx, d_k, sgd, nodes, node_w)
        ctx.gather_rows(Xpar, nodes.data_ptr(), Xs, n_pad)
        if Ls is not None:
            ctx.gather_rows(Lpar, nodes.data_ptr(), Ls, n_pad)
        runner.forward_backward(sgd, Xs, labels=labels, dH_top=dH, node_w=node_w if cfg.head != "none" else None)

    def run_batch(b, timed):
        """Sample one batch, capture the step, replay it P times; returns (work, sampler ms)."""
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        batch = pg.sample(cfg.n, cfg.m, seed0 + b * P, count=P)
        e.record(stream)
        work = 0
        for k in range(P):
            info = batch.get(k)
            work += runner.work_edge_features(info["nnz"] + info["n"])
        with torch.cuda.stream(stream):
            d_k.zero_()
            if not timed:
                one(batch)  # eager warm-up: workspaces grow outside any capture
                d_k.zero_()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            one(batch)
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            r0.record(stream)
            for _ in range(P):
                g.replay()
            r1.record(stream)
        stream.synchronize()
        batch.check()
        samp = a.elapsed_time(e)
        replay_ms[0] += r0.elapsed_time(r1)
        del g
        batch.free()
        return work, samp

    replay_ms = [0.0]
    run_batch(0, False)  # warm-up batch
    replay_ms[0] = 0.0
    nb = max(1, args.sampler_batches)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record(stream)
    work, samp_ms = 0, 0.0
    for b in range(1, nb + 1):
        w, sm = run_batch(b, True)
        work += w
        samp_ms += sm
    t1.record(stream)
    stream.synchronize()
    ms = t0.elapsed_time(t1)
    steps = nb * P
    sgd.free()
    pg.free()
    return {"value": work / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "subgraphs_per_gpu_sampler_call": P, "sampler_ms_per_subgraph": samp_ms / steps,
            "sampler_share": samp_ms / ms, "launch_mode": "one CUDA graph per sampled batch (gsg_sample_load)",
            "replay_ms_per_step": replay_ms[0] / steps,
            "note": "fresh GPU-sampled subgraph every step; the timed region includes the sampling calls "
                    "(gsg_frontier_sample, host-synchronized), the graph capture per batch and every replay"}


# ------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pool", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly instead of a CUDA graph")
    ap.add_argument("--no-comm-overlap", action="store_true",
                    help="issue the gradient all-reduce on the compute stream after each step (default: on a "
                         "communication stream, overlapping the next step's forward)")
    ap.add_argument("--no-relu-bits", action="store_true",
                    help="gate the backward with the fp32 activations instead of their ReLU bitmasks (A/B)")
    ap.add_argument("--nccl-self", action="store_true",
                    help="N = 1: build a 1-rank NCCL communicator so the all-reduce path (a9) runs and is timed")
    ap.add_argument("--batch", type=int, default=1,
                    help="B independent subgraphs per step as one block-diagonal graph (SURVEY §8(d) batched variant)")
    ap.add_argument("--sampler", default="host", choices=["host", "gpu"],
                    help="gpu: additionally time a training loop whose subgraphs are frontier-sampled on the GPU "
                         "(NEXT #3) from a device-resident parent graph, features gathered from a parent feature "
                         "matrix in HBM, a fresh subgraph every step")
    ap.add_argument("--sampler-pool", type=int, default=888,
                    help="subgraphs per GPU sampling call (--sampler gpu; 6 per SM keep the latency-bound samplers busy)")
    ap.add_argument("--sampler-batches", type=int, default=2,
                    help="timed sampling calls of --sampler gpu (each followed by --sampler-pool graph replays)")
    ap.add_argument("--nccl-timeout-ms", type=int, default=300000,
                    help="gsg_nccl_wait time-out for the all-reduce (a stalled or dead peer aborts the run)")
    ap.add_argument("--flush-l2", action="store_true",
                    help="flush L2 (write a 2x-L2 buffer) before every step of the per-step timing pass")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = wl.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2010_03166_b200 as gsg
    from paper_2010_03166_b200 import dp
    from paper_2010_03166_b200.step import GCNStep

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        with stdout_to_stderr():
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    t_setup = time.time()

    # ---- host inputs (seeded; outside every timed region) ----
    if args.batch > 1:
        pool = [wl.sample_batch(cfg, args.batch, k, rank) for k in range(args.pool)]
    else:
        pool = [wl.sample_subgraph(cfg, k, rank) for k in range(args.pool)]
    inputs = [wl.make_inputs(cfg, g.n, k, rank) for k, g in enumerate(pool)]
    n_max = max(g.n for g in pool)

    stream = torch.cuda.Stream(device=dev)
    ctx = gsg.Context(local, stream)
    with torch.cuda.stream(stream):
        sgs = [ctx.upload(g.indptr, g.indices, validate=True) for g in pool]
        f0 = cfg.dims[0]
        Xd = [torch.zeros((n_max, wl.ld_for(f0)), device=dev)[:, :f0] for _ in pool]
        for x, inp in zip(Xd, inputs):
            x[:inp.X.shape[0]].copy_(torch.from_numpy(inp.X))
        if cfg.head == "softmax":
            labd = [torch.from_numpy(inp.labels).to(dev) for inp in inputs]
        elif cfg.head == "sigmoid":
            labd = [torch.from_numpy(inp.labels).to(dev) for inp in inputs]
        else:
            labd = [None for _ in inputs]
        dHd = [None if inp.dH is None else torch.zeros((n_max, wl.ld_for(cfg.dims[-1])), device=dev)[:, :cfg.dims[-1]]
               for inp in inputs]
        for t, inp in zip(dHd, inputs):
            if t is not None:
                t[:inp.dH.shape[0]].copy_(torch.from_numpy(inp.dH))
        runner = GCNStep(ctx, cfg.dims, n_max, cfg.head, cfg.classes, cfg.precision, device=local,
                         weights=inputs[0].Ws, w_mlp=inputs[0].W_mlp, relu_bits=not args.no_relu_bits)
    stream.synchronize()
    comm = None
    if world > 1 or args.nccl_self:
        with stdout_to_stderr():
            uid = dp.broadcast_bytes(ctx.nccl_unique_id() if rank == 0 else None)
            comm = ctx.nccl_comm_init(world, rank, uid)
    # a9 overlap: the all-reduce of step i runs on a communication stream while step i+1 runs its
    # forward; the replayed step waits for it (external event node) right before it writes the
    # gradients again (GCNStep before_grads)
    overlap = comm is not None and not args.no_comm_overlap and not args.no_graph
    comm_stream = comm_ctx = ev_step = ev_ar = None
    if overlap:
        comm_stream = torch.cuda.Stream(device=dev)
        comm_ctx = gsg.Context(local, comm_stream)
        ev_step, ev_ar = torch.cuda.Event(), torch.cuda.Event()
        ev_ar.record(comm_stream)  # creates the event (an unrecorded wait would be a no-op anyway)

    nnz_hat = [g.nnz + g.n for g in pool]
    nnz_raw = [g.nnz for g in pool]
    act_bytes = 4 * n_max * sum(cfg.dims) * 4  # X/P/H/dX-class buffers per step, lower bound
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    l2_note = (f"step working set (>= {act_bytes / 1e6:.0f} MB of activations) exceeds the {l2_bytes / 1e6:.0f} MB L2; "
               f"{len(pool)} subgraphs rotate" if act_bytes > l2_bytes else
               f"step working set ({act_bytes / 1e6:.0f} MB) fits the {l2_bytes / 1e6:.0f} MB L2: warm-cache numbers; "
               "step_ms_dist with --flush-l2 gives the flushed figure")

    def step(i, with_comm=True, wait_ar=False, input_grad=True):
        k = i % len(pool)
        n = pool[k].n
        runner.forward_backward(sgs[k], Xd[k][:n], labels=labd[k], dH_top=None if dHd[k] is None else dHd[k][:n],
                                comm=comm if with_comm else None,
                                before_grads=(lambda: ctx.wait_event(ev_ar)) if wait_ar else None,
                                input_grad=input_grad)
        return runner.work_edge_features(nnz_hat[k], input_grad)

    # ---- normalize every pool slot once (grows its device arrays outside any graph capture) ----
    with torch.cuda.stream(stream):
        for sgk in sgs:
            sgk.normalize()
    stream.synchronize()

    # ---- warm-up (also JITs tensor maps / workspace growth) ----
    l0 = ctx.launch_count()
    for i in range(args.warmup):
        step(i)
    launches_per_step = (ctx.launch_count() - l0) / args.warmup
    stream.synchronize()

    # ---- one CUDA graph per pool slot: the whole step (normalize, L layers, head, backward,
    # all-reduce) captured once and replayed -- no per-kernel host launch cost in the loop ----
    graphs, graph_note = None, "eager"
    if not args.no_graph:
        try:
            graphs = []
            for k in range(len(pool)):
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph, stream=stream):
                    step(k, with_comm=False, wait_ar=overlap)  # a9 is issued after the replay
                graphs.append(gph)
            graph_note = "cuda-graph replay of the step (a1-a8) + eager NCCL all-reduce (a9)"
        except Exception as e:  # noqa: BLE001
            graphs, graph_note = None, f"eager (graph capture failed: {str(e)[:120]})"
            torch.cuda.synchronize()

    def step_run(i):
        if graphs is None:
            return step(i)
        k = i % len(pool)
        with torch.cuda.stream(stream):
            graphs[k].replay()
        if overlap:
            ev_step.record(stream)
            comm_stream.wait_event(ev_step)
            comm_ctx.allreduce_grads(comm, [runner.grad_flat], average=True)
            ev_ar.record(comm_stream)
        elif comm is not None:
            ctx.allreduce_grads(comm, [runner.grad_flat], average=True)
        return runner.work_edge_features(nnz_hat[k])

    def drain_comm():
        """The timed region ends when the last all-reduce has finished."""
        if overlap:
            stream.wait_event(ev_ar)

    def wait_stream():
        """stream.synchronize() with NCCL failure detection when a communicator exists
        (gsg_nccl_wait: asynchronous NCCL errors and a stall time-out abort the run loudly)."""
        if comm is not None:
            if comm_ctx is not None:
                comm_ctx.nccl_wait(comm, args.nccl_timeout_ms)
            ctx.nccl_wait(comm, args.nccl_timeout_ms)
        stream.synchronize()

    for i in range(2):
        step_run(i)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    # ---- timed region: inputs resident in HBM (no per-kernel instrumentation) ----
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count()
    work = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            work += step_run(i)
        drain_comm()
        ev1.record(stream)
        wait_stream()
    launches = int(round(launches_per_step * args.steps)) if graphs is not None else ctx.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    nccl_info = nccl_log_summary() if comm is not None else None
    # a9 alone: K back-to-back all-reduces of the flat gradient buffer on the stream the step uses
    ar_ms = None
    if comm is not None:
        ar_ctx, ar_stream = (comm_ctx, comm_stream) if overlap else (ctx, stream)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ar_stream.synchronize()
        a0.record(ar_stream)
        for _ in range(args.steps):
            ar_ctx.allreduce_grads(comm, [runner.grad_flat], average=True)
        a1.record(ar_stream)
        ar_ctx.nccl_wait(comm, args.nccl_timeout_ms)
        ar_ms = a0.elapsed_time(a1) / args.steps
    per_rank = {"rank": rank, "nnz_hat": nnz_hat, "nodes": [g.n for g in pool], "ms_per_step": ms / args.steps,
                "allreduce_ms": ar_ms, "allreduce_bytes": runner.grad_flat.numel() * 4}
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank)
        per_rank = gathered
    else:
        per_rank = [per_rank]
    torch.cuda.synchronize()
    max_ms, total_work = dp.reduce_timing(ms, float(work), device=dev)
    value = total_work / (max_ms / 1e3)
    # the same timed steps counted without self loops (nnz instead of nnz'), and in subgraphs/s
    work_noself = sum(runner.work_edge_features(nnz_raw[i % len(pool)]) for i in range(args.steps))
    _, total_noself = dp.reduce_timing(ms, float(work_noself), device=dev)
    value_noself = total_noself / (max_ms / 1e3)
    subgraphs_per_s = world * args.steps * args.batch / (max_ms / 1e3)

    # ---- training mode: the same step without layer 1's input gradient dX (which
    # training does not use), graph-replayed, all-reduce excluded; work counted without that a7 ----
    training = None
    if graphs is not None:
        try:
            tgraphs = []
            for k in range(len(pool)):
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph, stream=stream):
                    step(k, with_comm=False, input_grad=False)
                tgraphs.append(gph)
            te0, te1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                for i in range(2):
                    tgraphs[i % len(pool)].replay()
                te0.record(stream)
                for i in range(args.steps):
                    tgraphs[i % len(pool)].replay()
                te1.record(stream)
            stream.synchronize()
            tms = te0.elapsed_time(te1)
            twork = sum(runner.work_edge_features(nnz_hat[i % len(pool)], False) for i in range(args.steps))
            max_tms, total_twork = dp.reduce_timing(tms, float(twork), device=dev)
            training = {"ms_per_step": max_tms / args.steps, "value": total_twork / (max_tms / 1e3),
                        "unit": "edge_features/s",
                        "what": "step without layer 1's input gradient dX (SURVEY R6), graph replay, "
                                "all-reduce not included"}
            del tgraphs
        except Exception as e:  # noqa: BLE001
            torch.cuda.synchronize()
            training = {"unavailable": str(e)[:160]}

    # ---- the other GEMM precision beside the config's own (configs 1-2 run fp32-accurate 3xTF32
    # GEMMs; their plain-TF32 step is timed here as well, graph-replayed, all-reduce excluded) ----
    precision_alt = None
    if cfg.precision == "fp32x3" and graphs is not None:
        try:
            alt = GCNStep(ctx, cfg.dims, n_max, cfg.head, cfg.classes, "tf32", device=local,
                          weights=inputs[0].Ws, w_mlp=inputs[0].W_mlp, relu_bits=not args.no_relu_bits)
            agraphs = []
            with torch.cuda.stream(stream):
                for k in range(len(pool)):  # warm (workspace growth outside the capture)
                    alt.forward_backward(sgs[k], Xd[k][:pool[k].n], labels=labd[k],
                                         dH_top=None if dHd[k] is None else dHd[k][:pool[k].n])
            stream.synchronize()
            for k in range(len(pool)):
                gph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gph, stream=stream):
                    alt.forward_backward(sgs[k], Xd[k][:pool[k].n], labels=labd[k],
                                         dH_top=None if dHd[k] is None else dHd[k][:pool[k].n])
                agraphs.append(gph)
            ae0, ae1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                for i in range(2):
                    agraphs[i % len(pool)].replay()
                ae0.record(stream)
                for i in range(args.steps):
                    agraphs[i % len(pool)].replay()
                ae1.record(stream)
            stream.synchronize()
            ams, awork = dp.reduce_timing(ae0.elapsed_time(ae1),
                                          float(sum(alt.work_edge_features(nnz_hat[i % len(pool)])
                                                    for i in range(args.steps))), device=dev)
            precision_alt = {"precision": "tf32", "ms_per_step": ams / args.steps, "value": awork / (ams / 1e3),
                             "unit": UNIT, "what": "the same step with plain TF32 GEMMs (5e-3 parity) instead of "
                                                   "3xTF32 (1e-5), graph replay, all-reduce not included"}
            del agraphs, alt
        except Exception as e:  # noqa: BLE001
            torch.cuda.synchronize()
            precision_alt = {"unavailable": str(e)[:160]}

    # ---- per-step distribution: an event pair around every step (optionally after an L2 flush,
    # outside the bracket) -> p10 / p50 / p90 ms per step ----
    flush = None
    if args.flush_l2:
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
        evs[i][0].record(stream)
        step_run(i)
        evs[i][1].record(stream)
    stream.synchronize()
    per_step = sorted(a.elapsed_time(b) for a, b in evs)

    def pct(q):
        return per_step[min(len(per_step) - 1, int(round(q * (len(per_step) - 1))))]
    step_dist = {"p10": pct(0.1), "p50": pct(0.5), "p90": pct(0.9),
                 "l2": "flushed before every step" if flush is not None else "not flushed (working set vs L2 as in config.l2)"}

    # ---- the same K steps again with CUDA events around every launch (kernel-level rooflines):
    # captured in one CUDA graph with the event records as graph nodes and replayed once, so the
    # per-stage times carry no host launch gaps (eager fallback if capture fails) ----
    pv0, pv1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    drain_comm()  # the last overlapped all-reduce must finish before grad_flat is rewritten
    stream.synchronize()
    ctx.profile(True)
    prof_mode = "eager"
    if graphs is not None:
        try:
            pg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(pg, stream=stream):
                for i in range(args.steps):
                    step(i, with_comm=False)
            with torch.cuda.stream(stream):
                pv0.record(stream)
                pg.replay()
                pv1.record(stream)
            prof_mode = "graph"
        except Exception:  # noqa: BLE001
            torch.cuda.synchronize()
            for k in range(gsg.GSG_K_CLASSES):
                ctx.profile_read(k)  # drop the partial records of the failed capture
    if prof_mode == "eager":
        pv0.record(stream)
        for i in range(args.steps):
            step(i)
        pv1.record(stream)
    stream.synchronize()
    prof = {name: ctx.profile_read(k) for name, k in
            (("spmm", gsg.GSG_K_SPMM), ("gemm", gsg.GSG_K_GEMM), ("normalize", gsg.GSG_K_NORM), ("other", gsg.GSG_K_OTHER))}
    row_names = (("a1_normalize", gsg.GSG_K_A1), ("a2_aggregate", gsg.GSG_K_A2), ("a3_transform", gsg.GSG_K_A3),
                 ("a4_gate", gsg.GSG_K_A4), ("a5_dW", gsg.GSG_K_A5), ("a6_T", gsg.GSG_K_A6),
                 ("a7_aggregate_T", gsg.GSG_K_A7), ("a8_head", gsg.GSG_K_A8))
    rows_prof = {name: ctx.profile_read(k) for name, k in row_names}
    ctx.profile(False)
    prof_ms = pv0.elapsed_time(pv1)

    # ---- end to end: same calls, inputs copied from pinned host memory every step ----
    e2e = None
    if not args.no_e2e:
        pin_ip = [torch.from_numpy(g.indptr).pin_memory() for g in pool]
        pin_ix = [torch.from_numpy(g.indices).pin_memory() for g in pool]
        pin_X = [torch.from_numpy(np.ascontiguousarray(inp.X)).pin_memory() for inp in inputs]
        pin_lab = [None if inp.labels is None else torch.from_numpy(inp.labels).pin_memory() for inp in inputs]
        pin_dH = [None if inp.dH is None else torch.from_numpy(inp.dH).pin_memory() for inp in inputs]
        loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()
        h2d = 0

        # Double-buffered input slots (the pool's two subgraph/X/label slots): the copies of step
        # i+1's inputs run on a copy stream while step i computes; step i+1 waits for them, and a
        # slot is refilled only after the step that last read it has finished.
        cstream = torch.cuda.Stream(device=dev)
        cctx = gsg.Context(local, cstream)
        copied = [torch.cuda.Event() for _ in pool]
        consumed = [torch.cuda.Event() for _ in pool]
        for k in range(len(pool)):
            consumed[k].record(stream)
        step_bytes = []
        for k, g in enumerate(pool):
            b = pin_ip[k].numel() * 8 + pin_ix[k].numel() * 4 + pin_X[k].numel() * 4
            b += 0 if pin_lab[k] is None else pin_lab[k].numel() * pin_lab[k].element_size()
            b += 0 if pin_dH[k] is None else pin_dH[k].numel() * 4
            step_bytes.append(b)

        def issue_copy(i):
            k = i % len(pool)
            g = pool[k]
            cstream.wait_event(consumed[k])
            sgs[k].assign(g.n, g.nnz, pin_ip[k].data_ptr(), pin_ix[k].data_ptr(), ctx=cctx)
            with torch.cuda.stream(cstream):
                Xd[k][:g.n].copy_(pin_X[k], non_blocking=True)
                if labd[k] is not None:
                    labd[k].copy_(pin_lab[k], non_blocking=True)
                if dHd[k] is not None:
                    dHd[k][:g.n].copy_(pin_dH[k], non_blocking=True)
            copied[k].record(cstream)

        def run_e2e(n_steps, start_event=None):
            nonlocal h2d
            work = 0
            if start_event is not None:
                cstream.wait_event(start_event)
            issue_copy(0)
            for i in range(n_steps):
                k = i % len(pool)
                if i + 1 < n_steps:
                    issue_copy(i + 1)
                stream.wait_event(copied[k])
                work += step_run(i)
                consumed[k].record(stream)
                with torch.cuda.stream(stream):
                    loss_host.copy_(runner.loss, non_blocking=True)
                h2d = step_bytes[k]
            return work

        run_e2e(args.warmup)
        stream.synchronize()
        cstream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ework = run_e2e(args.steps, start_event=e0)
        drain_comm()
        e1.record(stream)
        stream.synchronize()
        ems, ework_all = dp.reduce_timing(e0.elapsed_time(e1), float(ework), device=dev)
        e2e = {"value": ework_all / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4,
               "ms_per_step": ems / args.steps, "loss": float(loss_host.item())}

    # ---- roofline of the dominant kernel (the SpMM, a2 + a7) ----
    # X is L2-resident (<= 82 MB of the 126 MB L2), so the kernel's binding ceiling is the L2->SM
    # random-gather rate, measured here in the same run (gsg_diag_gather_ceiling: whole-row
    # gathers at random row ids from this step's own activation matrix); DRAM is reported apart
    # (minimum-HBM bytes, and the ncu DRAM traffic of this config's launches where captured).
    peaks = load_peaks()
    sp = prof["spmm"]
    spmm_gbs = sp["alg_bytes"] / (sp["ms"] / 1e3) / 1e9 if sp["ms"] > 0 else 0.0
    widths = runner.spmm_widths()
    wide_l = max(range(cfg.L), key=lambda l: cfg.dims[l + 1])
    probe_src = runner.H[wide_l]
    ceil_by_row = {}
    for f_probe, src in ((min(256, cfg.dims[wide_l + 1]) // 8 * 8, probe_src),
                         (min(256, cfg.dims[0]) // 8 * 8, Xd[0])):
        if f_probe >= 8 and str(f_probe * 4) not in ceil_by_row:
            ceil_by_row[str(f_probe * 4)] = ctx.diag_gather_ceiling(src, f_probe)
    probe_row_bytes = min(256, cfg.dims[wide_l + 1]) // 8 * 8 * 4
    l2_ceiling = ceil_by_row[str(probe_row_bytes)]
    n_avg = sum(g.n for g in pool) / len(pool)
    nh_avg = sum(nnz_hat) / len(pool)
    min_hbm_step = sum(8 * nh_avg + 4 * (n_avg + 1) + 8 * n_avg * f for f in widths)
    eff_step = sp["alg_bytes"] / args.steps
    sp_ms_step = sp["ms"] / args.steps
    dram = None
    tpath = os.path.join(ROOT, "profiles", f"spmm_traffic_c{cfg.cid}.json")
    if os.path.exists(tpath) and args.batch == 1:
        with open(tpath) as f:
            td = json.load(f)
        byw = td.get("dram_bytes_by_width", {})
        if td.get("config") == cfg.cid and all(str(f) in byw for f in widths):
            dram_step = sum(byw[str(f)] for f in widths)
            min_w = {str(f): 8 * nh_avg + 4 * (n_avg + 1) + 8 * n_avg * f for f in set(widths)}
            dram = {"bytes_per_step": dram_step, "bytes_per_launch": dram_step / len(widths),
                    "by_width": {f: {"dram_bytes": byw[f], "min_hbm_bytes": min_w[f], "dram_over_min": byw[f] / min_w[f]}
                                 for f in sorted(min_w, key=int)},
                    "source": f"{os.path.relpath(tpath, ROOT)} (ncu dram__bytes_read.sum + dram__bytes_write.sum of one "
                              f"config-{cfg.cid} step's SpMM launches)"}
    roofline = {"bound": "l2", "achieved": spmm_gbs, "peak": l2_ceiling, "unit": "GB/s",
                "frac": spmm_gbs / l2_ceiling if l2_ceiling else None,
                "traffic": None if dram is None else dram["bytes_per_launch"],
                "kernel": "k_spmm (a2 P=ÂX and a7 dX=ÂᵀT), algorithmic effective gather bytes "
                          "(4·nnz'·f + 8·nnz' + 4(n+1) + 4·n·f per launch) / kernel time",
                "peak_source": f"measured in this run: gsg_diag_gather_ceiling, random {probe_row_bytes}-byte "
                               f"row gathers from this step's {n_max}x{cfg.dims[wide_l + 1]} activation matrix "
                               "(L2-resident), best of 2/3/4 CTAs per SM",
                "peak_by_row_bytes": ceil_by_row,
                "hbm": {"min_bytes_per_step": min_hbm_step, "achieved_gbs": min_hbm_step / (sp_ms_step / 1e3) / 1e9,
                        "peak": peaks["hbm_gbs"], "frac": min_hbm_step / (sp_ms_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks['source']})",
                        "note": "minimum-HBM bytes (X read once: 8·nnz' + 4(n+1) + 8·n·f per launch) over the SpMM "
                                "time; the SpMM is not DRAM-bound (X is L2-resident)",
                        "dram_traffic": dram,
                        "effective_over_hbm_peak": spmm_gbs / peaks["hbm_gbs"]},
                "effective_bytes_per_step": eff_step, "widths_per_step": widths,
                "launches": sp["launches"], "kernel_ms": sp["ms"],
                "share_of_step": sp["ms"] / prof_ms if prof_ms > 0 else None,
                "timing": f"per-launch CUDA events on the launch stream, second ({prof_mode}-replayed) pass of the "
                          "same K steps"}
    gm = prof["gemm"]
    tf32_peak = peaks["bf16_tflops"] / 2.0  # TF32 = 1/2 of the measured BF16 burst peak (nominal ratio)
    gemm_tflops = gm["alg_flops"] / (gm["ms"] / 1e3) / 1e12 if gm["ms"] > 0 else 0.0
    gemm_info = {"bound": "tensor", "achieved": gemm_tflops, "unit": "TFLOP/s",
                 "peak": tf32_peak if cfg.precision != "bf16" else peaks["bf16_tflops"],
                 "peak_note": ("measured bf16 burst x 1/2 (nominal TF32:BF16)" if cfg.precision != "bf16"
                               else "measured bf16 burst") +
                              ("; fp32x3 flops counted as executed on the TF32 pipe (3 per product)"
                               if cfg.precision == "fp32x3" else ""),
                 "kernel_ms": gm["ms"], "launches": gm["launches"],
                 "share_of_step": gm["ms"] / prof_ms if prof_ms > 0 else None}
    gemm_info["frac"] = gemm_tflops / gemm_info["peak"]
    # Layer-level roofline fraction: ideal step time from the algorithmic totals --
    # SpMM effective bytes at a memory ceiling + GEMM flops at the tensor peak + the other
    # kernels' bytes at HBM -- over the measured step time. Against HBM (the contract's number,
    # > 1 because X is L2-resident) and against the measured L2 random-gather ceiling.
    step_ms = max_ms / args.steps
    other_bytes = (prof["normalize"]["alg_bytes"] + prof["other"]["alg_bytes"]) / args.steps
    gemm_ideal_ms = gm["alg_flops"] / args.steps / (gemm_info["peak"] * 1e12) * 1e3
    other_ideal_ms = other_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3
    sp_bytes = sp["alg_bytes"] / args.steps
    layer_roof = {"hbm": (sp_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3 + gemm_ideal_ms + other_ideal_ms) / step_ms}
    if l2_ceiling:
        layer_roof["l2_gather"] = (sp_bytes / (l2_ceiling * 1e9) * 1e3 + gemm_ideal_ms + other_ideal_ms) / step_ms
    layer_roof["note"] = ("(SpMM effective bytes / memory ceiling + GEMM flops / tensor peak + other bytes / HBM) "
                          "/ measured step time")

    # ---- CPU baseline: the oracle on host cores (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        osamp = OracleSample(cfg, pool[0], inputs[0])
        w_, dt_ = osamp.calibrate(args.cpu_seconds)
        cpu = {"value": w_ / dt_, "unit": UNIT, "cores": osamp.cores(), "kind": "oracle", "cpu_model": osamp.cpu_model(),
               "sample": f"rows [0,{osamp.rows}) of the first subgraph, all {cfg.L} layers fwd+bwd + head, "
                         f"fp64 plain loops, {dt_:.1f} s"}

    # ---- optional: the same step fed by the GPU sampler (a fresh subgraph every step) ----
    gpu_loop = None
    if args.sampler == "gpu" and args.batch == 1:
        # thousands of back-to-back steps: the clocks show whether the power cap engaged (compare
        # with a pooled run of similar length, e.g. --steps 1000)
        with ClockSampler(local) as clk_loop:
            gpu_loop = run_gpu_sampled(args, cfg, ctx, runner, stream, dev, rank, max(nnz_raw))
        gpu_loop["clocks"] = clk_loop.summary()

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": {"tf32": "f32 (SpMM) + tf32 (GEMM)", "bf16": "f32 (SpMM) + bf16 (GEMM)",
                                                     "fp32x3": "f32 (SpMM) + f32 via 3xtf32 (GEMM)"}[cfg.precision],
               "data": "synthetic",
               "config": {"workload": f"config{cfg.cid}:{cfg.name}" + (f" x{args.batch} block-diagonal batch"
                                                                         if args.batch > 1 else ""),
                          "nodes_per_gpu": max(g.n for g in pool), "subgraphs_per_step": args.batch,
                          "nnz_hat_per_gpu": nnz_hat, "dims": cfg.dims, "head": f"{cfg.head}{cfg.classes}",
                          "parent": {"n": cfg.parent_n, "mean_deg": cfg.parent_mean_deg, "gamma": cfg.gamma},
                          "pool_per_gpu": len(pool), "parallelism": f"dp{world}",
                          "allreduce": ("none" if comm is None else
                                        "overlapped with the next step's forward (comm stream)" if overlap else
                                        "after each step on the compute stream"),
                          "relu_gate": "fp32 activations" if args.no_relu_bits else "bitmask",
                          "l2": l2_note},
               "roofline": roofline, "gemm": gemm_info, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "launch_mode": graph_note, "clocks": clk.summary(),
               "stages_ms_per_step": {k: v["ms"] / args.steps for k, v in prof.items()},
               "rows_ms_per_step": {k: v["ms"] / args.steps for k, v in rows_prof.items()},
               "stage_timing": f"per-launch CUDA events ({prof_mode} pass of the same steps, dW GEMM not forked "
                               "while profiling); ms_per_step is the graph-replayed step",
               "step_ms_dist": step_dist, "training_mode": training,
               "value_noself": value_noself, "subgraphs_per_s": subgraphs_per_s,
               "layer_roofline_frac": layer_roof,
               "per_rank": per_rank, "nccl": nccl_info, "precision_alt": precision_alt,
               "setup_s": time.time() - t_setup}
        if gpu_loop is not None:
            out["gpu_sampled_loop"] = gpu_loop
        print(json.dumps(out), flush=True)
    if comm is not None:
        stream.synchronize()
        ctx.nccl_comm_destroy(comm)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
