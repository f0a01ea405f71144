mkdir -p gpurun_out/sweep2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_k.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_k.log
timeout 600 python bench.py > gpurun_out/sweep2/c5.json 2> gpurun_out/sweep2/c5.err; echo c5=$?
for c in 1 2 3 4; do timeout 600 python bench.py --config $c --no-cpu --steps 50 > gpurun_out/sweep2/c$c.json 2> gpurun_out/sweep2/c$c.err; echo c$c=$?; done
timeout 600 python bench.py --config 1 --no-cpu --steps 50 --flush-l2 > gpurun_out/sweep2/c1_flush.json 2> gpurun_out/sweep2/c1_flush.err; echo c1f=$?
timeout 600 python bench.py --config 1 --no-cpu --steps 50 --batch 64 > gpurun_out/sweep2/c1_b64.json 2> gpurun_out/sweep2/c1_b64.err; echo c1b=$?
timeout 600 python bench.py --config 5 --no-cpu --steps 32 --pool 8 --no-e2e > gpurun_out/sweep2/c5_pool8.json 2> gpurun_out/sweep2/c5_pool8.err; echo c5p8=$?
timeout 600 python bench.py --config 5 --no-cpu --steps 30 --no-e2e --flush-l2 > gpurun_out/sweep2/c5_flush.json 2> gpurun_out/sweep2/c5_flush.err; echo c5f=$?
timeout 900 python tools/oracle_timing.py > gpurun_out/sweep2/oracle.jsonl 2> gpurun_out/sweep2/oracle.err; echo orc=$?
OMP_NUM_THREADS=1 timeout 300 python tools/oracle_timing.py 1 >> gpurun_out/sweep2/oracle.jsonl 2>> gpurun_out/sweep2/oracle.err; echo orc1=$?
nproc; lscpu | head -20 > gpurun_out/sweep2/lscpu.txt
