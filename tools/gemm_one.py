"""Measurement tool: one gsg_gemm shape, ITERS calls captured in a CUDA graph and replayed (device
time per call without host launch gaps; GRAPH=0 launches eagerly, e.g. under ncu).
SHAPE = "M,N,K,transA,transB", PREC = tf32 | bf16, EPI = none | relu | relubits | mask | maskbits."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_03166_b200 as gsg  # noqa: E402


def main():
    M, N, K, ta, tb = (int(x) for x in os.environ.get("SHAPE", "20000,1024,200,0,0").split(","))
    prec = gsg.GSG_PREC_BF16 if os.environ.get("PREC", "tf32") == "bf16" else gsg.GSG_PREC_TF32
    epi = os.environ.get("EPI", "none")
    iters = int(os.environ.get("ITERS", "20"))
    tdt = torch.bfloat16 if prec == gsg.GSG_PREC_BF16 else torch.float32

    def pad(r, c, dt=tdt):
        return torch.randn((r, (c + 7) // 8 * 8), device="cuda", dtype=dt)[:, :c]
    A = pad(*((K, M) if ta else (M, K)))
    B = pad(*((N, K) if tb else (K, N)))
    C = torch.empty((M, (N + 7) // 8 * 8), device="cuda")[:, :N]
    kw = {}
    if epi == "relu":
        kw["epilogue"] = gsg.GSG_EPI_RELU
    elif epi == "mask":
        kw["epilogue"] = gsg.GSG_EPI_MASK
        kw["aux"] = pad(M, N, torch.float32)
    elif epi == "maskbits":  # ReLU' gate from a bitmask (as the step's dH_L GEMM)
        kw["epilogue"] = gsg.GSG_EPI_MASK
        kw["aux_bits"] = torch.randint(-2**31, 2**31 - 1, (M, (N + 31) // 32), dtype=torch.int32, device="cuda")
    elif epi == "relubits":  # ReLU epilogue that also writes the bitmask (as the step's forward GEMMs)
        kw["epilogue"] = gsg.GSG_EPI_RELU
        kw["C_bits"] = torch.zeros((M, (N + 31) // 32), dtype=torch.int32, device="cuda")
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    graph = os.environ.get("GRAPH", "1") == "1"

    def run():
        ctx.gemm(A, B, C, transA=bool(ta), transB=bool(tb), precision=prec, K=K, **kw)
    with torch.cuda.stream(stream):
        for _ in range(3):
            run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(iters):
                run()
        g.replay()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            a.record()
            g.replay()
            b.record()
    else:
        with torch.cuda.stream(stream):
            a.record()
            for _ in range(iters):
                run()
            b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / iters * 1e3
    print(f"SHAPE={M},{N},{K},{ta},{tb} PREC={os.environ.get('PREC', 'tf32')} EPI={epi}: {us:.2f} us/call "
          f"{2.0 * M * N * K / us / 1e6:.1f} TFLOP/s ({'graph replay' if graph else 'eager'})")


if __name__ == "__main__":
    main()
