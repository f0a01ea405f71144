timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_o.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_o.log
for so in 0 1; do for si in 0 1; do
  GSG_SPMM_STREAM_OUT=$so GSG_SPMM_STREAM_IN=$si WIDTHS=200,1024 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{' | sed "s/^/out$so in$si /"
  GSG_SPMM_STREAM_OUT=$so GSG_SPMM_STREAM_IN=$si timeout 300 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_o$so$si.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_o$so$si.json'));print('out$so in$si bench', d['ms_per_step'], d['stages_ms_per_step'])"
done; done
