"""Measurement tool (SURVEY §8(d) "Oracle timing", reported baseline only): the fp64 oracle
as it stands, on the host cores, for every config -- a bounded row sample of one full
forward + backward step (bench.OracleSample) -- and config 1's whole step as the serial point
when run with OMP_NUM_THREADS=1. One JSON line per config.

    python tools/oracle_timing.py [configs...]            # default 1 2 3 4 5
    OMP_NUM_THREADS=1 python tools/oracle_timing.py 1     # serial point
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import workload as wl  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    cids = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]
    budget = float(os.environ.get("ORACLE_SECONDS", "8"))
    for c in cids:
        cfg = wl.CONFIGS[c]
        g = wl.sample_subgraph(cfg, 0, 0)
        inp = wl.make_inputs(cfg, g.n, 0, 0)
        osamp = bench.OracleSample(cfg, g, inp)
        t0 = time.perf_counter()
        if c == 1:
            osamp.run(g.n)  # warm (thread pool, page faults)
            work, dt = min((osamp.run(g.n) for _ in range(3)), key=lambda r: r[1])
        else:
            work, dt = osamp.calibrate(budget)
        full = osamp.rows is None or osamp.rows == g.n
        print(json.dumps({"config": c, "n": g.n, "nnz_hat": g.nnz + g.n, "rows_timed": osamp.rows or g.n,
                          "full_step": full, "seconds": dt, "edge_features_per_s": work / dt,
                          "threads": bench.OracleSample.cores(), "cpu": cpu_model(),
                          "wall_incl_calibration_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
