timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_b.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_b.log
for a in 8 32; do LD_ALIGN=$a WIDTHS=200,300,602,1024 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{'; done | tee gpurun_out/ld_ab.jsonl
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_b.json 2>gpurun_out/bench_b.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_b.json'));print(d['ms_per_step'], d['stages_ms_per_step'], d['step_ms_dist'])"
