"""bench.py's reference arm needs no GPU (it times the fp64 oracle on the host cores): its JSON
line is checked here, in the CPU suite, on a short config-1 run, together with the torchrun rule
that only rank 0 runs it (other ranks exit 0 without output)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(env_extra=None, *args):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=env)


def test_reference_arm_line_on_cpu():
    out = run(None, "--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["dtype"] == "f64" and d["steps"] == 1
    assert d["metric"] and d["unit"] and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert cb["cpu_model"]  # the host CPU is named (BASELINE.md plan item 3)
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("config1")


def test_reference_arm_other_ranks_exit_quietly():
    out = run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--impl", "reference", "--config", "1",
              "--steps", "1", "--warmup", "3")
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == ""


def test_nccl_log_summary(tmp_path, monkeypatch, capsys):
    """bench.py's NCCL INFO log handling: copied to stderr (not stdout, which carries only the JSON
    line) and summarized (ranks NCCL saw, NVLS set-up lines)."""
    import importlib.util
    log = tmp_path / "nccl.log"
    log.write_text("h:1:1 [0] NCCL INFO NCCL version 2.28.9+cuda12.9\n"
                   "h:1:1 [0] NCCL INFO comm 0x1 rank 0 nRanks 8 nNodes 1 localRanks 8 localRank 0 MNNVL 0\n"
                   "h:1:1 [0] NCCL INFO NVLS multicast support is available on dev 0 (NVLS_NCHANNELS 16)\n")
    monkeypatch.setenv("NCCL_DEBUG_FILE", str(log))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    s = bench.nccl_log_summary()
    cap = capsys.readouterr()
    assert cap.out == "" and "nRanks 8" in cap.err
    assert s["nranks_seen"] == [8] and s["nvls"] and s["version"].startswith("2.28.9")
