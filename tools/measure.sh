#!/usr/bin/env bash
# How the round's GPU evidence under profiles/ is produced (run on a B200 box, e.g. through
# gpurun, from the repo root). Each step only after the previous command exited 0 without ncu.
set -x
mkdir -p gpurun_out/sweep
python -m pytest tests -m gpu -x -q                                   # parity suite
python bench.py > gpurun_out/sweep/c5.json                            # the driver's default line
for c in 1 2 3 4; do python bench.py --config $c --no-cpu --steps 50 > gpurun_out/sweep/c$c.json; done
python bench.py --config 1 --no-cpu --steps 50 --flush-l2 > gpurun_out/sweep/c1_flush.json
python bench.py --config 1 --no-cpu --steps 50 --batch 64 > gpurun_out/sweep/c1_b64.json
python bench.py --config 5 --no-cpu --steps 32 --pool 8 --no-e2e > gpurun_out/sweep/c5_pool8.json
python bench.py --config 5 --no-cpu --steps 30 --no-e2e --flush-l2 > gpurun_out/sweep/c5_flush.json
python tools/oracle_timing.py > gpurun_out/sweep/oracle.jsonl
OMP_NUM_THREADS=1 python tools/oracle_timing.py 1 >> gpurun_out/sweep/oracle.jsonl
python tools/gemm_bench.py > gpurun_out/gemm_bench.json               # ours vs cuBLAS, graph-replayed
WIDTHS=200,300,512,602,1024 python tools/spmm_bench.py                # SpMM alone per width
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2bw tools/l2bw.cu && tools/l2bw
# launch list of the bench step (shares, not absolutes: cold cache, serialized)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e
# one full capture of the top kernel (and of a big GEMM)
WIDTHS=1024 ncu --set full --import-source on --clock-control none -k regex:k_spmm_wide -s 2 -c 1 -f \
    -o gpurun_out/spmm1024 python tools/spmm_bench.py
SHAPE=20000,1024,1024,0,0 EPI=relu GRAPH=0 ITERS=4 ncu --set full --import-source on --clock-control none \
    -k regex:k_gemm -s 3 -c 1 -f -o gpurun_out/gemm1024 python tools/gemm_one.py
# summaries for profiles/ (here or on the CPU side)
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches_summary.json
python tools/ncu_summary.py report gpurun_out/spmm1024.ncu-rep gpurun_out/gemm1024.ncu-rep > gpurun_out/ncu_summary.json
