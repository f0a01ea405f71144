"""Measurement tool: our tcgen05 GEMM (gsg_gemm) vs cuBLAS (torch.matmul, TF32 / BF16) on the
config-5 GEMM shapes, plus the cuBLAS TF32 / BF16 peak on 8192^3 (burst). One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_03166_b200 as gsg  # noqa: E402


def timeit(fn, iters=20, warm=3, stream=None):
    """Device time per call. With a stream, the calls are captured in one CUDA graph and
    replayed, so host-side launch cost (tensor-map encoding, ctypes) is excluded."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if stream is not None:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            a.record()
            g.replay()
            b.record()
    else:
        a.record()
        for _ in range(iters):
            fn()
        b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    out = {}
    for dt, name in ((torch.float32, "tf32"), (torch.bfloat16, "bf16")):
        x = torch.randn(8192, 8192, device="cuda", dtype=dt)
        ms = timeit(lambda: x @ x, iters=10)
        out[f"cublas_{name}_8192_tflops"] = 2 * 8192 ** 3 / ms / 1e9
    stream = torch.cuda.Stream()
    ctx = gsg.Context(0, stream)
    n, f = 20000, 1024
    shapes = {
        "Z=P@W (K,MN)": (n, f, f, False, False),
        "dW=P^T@dZ (MN,MN)": (f, f, n, True, False),
        "T=dZ@W^T (K,K)": (n, f, f, False, True),
        "layer1 Z (K=200)": (n, f, 200, False, False),
        "layer1 T (N=200)": (n, 200, f, False, True),
        "head dHL (K=107)": (n, f, 107, False, True),
        "layer1 dW (M=200)": (200, f, n, True, False),
        "head S (N=107)": (n, 107, f, False, False),
    }
    for prec, tdt in ((gsg.GSG_PREC_TF32, torch.float32), (gsg.GSG_PREC_BF16, torch.bfloat16)):
        for label, (M, N, K, ta, tb) in shapes.items():
            def pad(r, c):
                return torch.randn((r, (c + 7) // 8 * 8), device="cuda", dtype=tdt)[:, :c]
            A = pad(*((K, M) if ta else (M, K)))
            B = pad(*((N, K) if tb else (K, N)))
            ldc = (N + 7) // 8 * 8
            C = torch.empty((M, ldc), device="cuda")[:, :N]
            flops = 2.0 * M * N * K
            ms = timeit(lambda: ctx.gemm(A, B, C, transA=ta, transB=tb, precision=prec, K=K), stream=stream)
            Am = A.t() if ta else A
            Bm = B.t() if tb else B
            ms_cub = timeit(lambda: torch.matmul(Am, Bm))
            key = f"{'tf32' if prec == 0 else 'bf16'} {label}"
            out[key] = {"ours_tflops": flops / ms / 1e9, "cublas_tflops": flops / ms_cub / 1e9, "ours_us": ms * 1e3}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
