#!/usr/bin/env bash
# How the round's GPU evidence under profiles/ is produced (run on a B200 box, e.g. through
# gpurun, from the repo root). Each step only after the previous command exited 0 without ncu.
# Output goes to gpurun_out/sweep_<tag>/; the summaries are copied into profiles/ by hand.
set -x
T=${TAG:-r02}
O=gpurun_out/sweep_$T
mkdir -p $O
python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1   # parity suite
python bench.py > $O/c5.json 2> $O/c5.err                             # the driver's default line
for c in 1 2 3 4; do python bench.py --config $c --no-cpu --steps 50 > $O/c$c.json 2>/dev/null; done
python bench.py --config 1 --no-cpu --steps 50 --flush-l2 > $O/c1_flush.json 2>/dev/null
python bench.py --config 1 --no-cpu --steps 50 --batch 64 > $O/c1_b64.json 2>/dev/null
python bench.py --config 5 --no-cpu --steps 32 --pool 8 --no-e2e > $O/c5_pool8.json 2>/dev/null
python bench.py --config 5 --no-cpu --steps 30 --no-e2e --flush-l2 > $O/c5_flush.json 2>/dev/null
python bench.py --config 5 --no-cpu --steps 30 --no-e2e --nccl-self > $O/c5_nccl.json 2>$O/c5_nccl.err
python bench.py --impl reference > $O/ref.json 2>/dev/null
python tools/gemm_bench.py > $O/gemm_bench.json 2>&1                   # ours vs cuBLAS, graph-replayed
WIDTHS=200,300,512,602,1024 python tools/spmm_bench.py > $O/spmm_widths.jsonl 2>&1
python tools/step_gaps.py > $O/timeline_c5.txt 2>&1
for c in 2 3 4; do CFG=$c python tools/step_gaps.py > $O/timeline_c$c.txt 2>&1; done
python bench.py --steps 1000 --warmup 20 --no-cpu --no-e2e > $O/c5_long1000.json 2>/dev/null      # sustained (power cap)
python bench.py --sampler gpu --no-cpu --no-e2e --steps 20 > $O/c5_sampled_loop.json 2>/dev/null  # GPU-sampled loop
# launch list of the bench step (shares, not absolutes: cold cache, serialized)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
# one full capture of the top kernel (f = 1024 SpMM) and of the in-step f = 200 SpMM and a big GEMM
WIDTHS=1024 ncu --set full --import-source on --clock-control none -k regex:k_spmm_wide -s 2 -c 1 -f \
    -o $O/spmm1024 python tools/spmm_bench.py > $O/ncu_spmm.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_spmm_wide -s 10 -c 1 -f \
    -o $O/spmm_step python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/ncu_spmm_step.log 2>&1
SHAPE=20000,1024,1024,0,0 EPI=relubits GRAPH=0 ITERS=4 ncu --set full --import-source on --clock-control none \
    -k regex:k_gemm -s 3 -c 1 -f -o $O/gemm1024 python tools/gemm_one.py > $O/ncu_gemm.log 2>&1
