"""Summarize ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>      per-kernel share of device time
  python tools/ncu_summary.py report <file.ncu-rep> [...]  key metrics of each captured launch
  python tools/ncu_summary.py traffic <spmm_metrics.csv> [cid]  DRAM / L2 bytes of the last step's
        SpMM launches, tagged by width -> profiles/spmm_traffic_c<cid>.json (bench.py's roofline.traffic)
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_op_hmma.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


DIAG = ("k_gather_probe",)  # measurement kernels of bench.py's roofline (gsg_diag_gather_ceiling), not the step


def launches(path):
    """Per-kernel share of the device time of the step's kernels (diagnostic probes excluded)."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in data:
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("ns", "nsecond") else (v * 1e3 if r[ui] in ("ms", "msecond") else v)
        name = re.sub(r"\(.*", "", r[ki])
        if any(d in name for d in DIAG):
            continue
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = []
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k, "launches": c, "total_us": round(t, 1), "avg_us": round(t / c, 2),
                    "share": round(t / tot, 4)})
    return {"total_us": round(tot, 1), "kernels": out}


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": re.sub(r"\(.*", "", r[h.index("Kernel Name")])}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def traffic(path, cid=5):
    """DRAM / L2 bytes of the last step's SpMM launches, each tagged with its feature width (the
    launch order of one step, paper_2010_03166_b200.step.spmm_widths) -> the per-config file
    bench.py reads (profiles/spmm_traffic_c<cid>.json)."""
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import workload as wl
    from paper_2010_03166_b200.step import chain_order, spmm_widths
    cfg = wl.CONFIGS[cid]
    widths = spmm_widths(cfg.dims, [chain_order(cfg.dims[l], cfg.dims[l + 1]) for l in range(cfg.L)])
    res = _traffic(path, len(widths))
    by_width = collections.OrderedDict()
    for x, f in zip(res["launches"], widths):
        x["f"] = f
        by_width.setdefault(str(f), []).append((x["dram_read"] or 0) + (x["dram_write"] or 0))
    res["config"] = cid
    res["widths"] = widths
    res["dram_bytes_by_width"] = {f: sum(v) / len(v) for f, v in by_width.items()}
    res["source"] = res["source"].replace("(one config-5 step)", f"(one config-{cid} step)")
    return res


def _traffic(path, k=6):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    idi, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
             "ms": 1e3, "msecond": 1e3}
    per = collections.OrderedDict()
    for r in data:
        per.setdefault(r[idi], {})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    ids = list(per)[-k:]
    out = []
    for j, i in enumerate(ids):
        m = per[i]
        out.append({"launch": j, "dram_read": m.get("dram__bytes_read.sum"), "dram_write": m.get("dram__bytes_write.sum"),
                    "lts_bytes": m.get("lts__t_bytes.sum"), "us": m.get("gpu__time_duration.sum")})
    tot = sum((x["dram_read"] or 0) + (x["dram_write"] or 0) for x in out)
    return {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum over the last {k} "
                      "k_spmm_* launches (one config-5 step) of bench.py --steps 2 --warmup 3",
            "launches": out, "dram_bytes_per_launch": tot / len(out) if out else None}


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "traffic":
        print(json.dumps(traffic(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 5), indent=1))
    elif mode == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps([x for p in sys.argv[2:] for x in report(p)], indent=1))
