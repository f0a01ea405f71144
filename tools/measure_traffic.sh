#!/usr/bin/env bash
# DRAM / L2 bytes of one step's SpMM launches per config (bench.py's roofline.traffic and
# roofline.hbm.dram_traffic read profiles/spmm_traffic_c<c>.json). Run on a B200 box; then here:
#   python tools/ncu_summary.py traffic gpurun_out/traffic_c<c>.csv <c> > profiles/spmm_traffic_c<c>.json
mkdir -p gpurun_out
for c in ${CFGS:-1 2 3 4 5}; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum \
      --clock-control none -k regex:k_spmm --csv \
      python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/traffic_c$c.csv 2>/dev/null
done
