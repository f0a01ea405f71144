"""Data-parallel step on >= 2 GPUs: runs
tests/workers/dp_nccl_worker.py under torchrun, one process per visible GPU (up to 8), and
checks gsg_allreduce_grads' mean against (a) the single-GPU dW for identical subgraphs (1e-6)
and (b) the mean of every rank's fp64 oracle dW for distinct subgraphs (5e-3). Skips with
fewer than 2 GPUs (the gpurun pool has one; the driver's 8-GPU tier runs it)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_dp_allreduce_multi_gpu(tmp_path):
    n = min(8, torch.cuda.device_count())
    out = tmp_path / "dp.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "workers", "dp_nccl_worker.py"), str(out)]
    env = dict(os.environ, NCCL_DEBUG="WARN")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    res = json.loads(out.read_text())
    assert len(res) == n
    for r in res:
        assert r["world"] == n
        assert r["identical_rel"] <= 1e-6, r
        assert r["distinct_rel"] <= 5e-3, r
        assert r["distinct_subgraphs"]
