timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "spmm or layer or sage" > gpurun_out/pytest_i.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_i.log
WIDTHS=200,1024 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{'
CFG=4 WIDTHS=200,1024 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{'
CFG=3 WIDTHS=300,512 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{'
CFG=2 WIDTHS=602,512 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{'
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_i.json 2>gpurun_out/bench_i.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_i.json'));print(d['ms_per_step'], d['stages_ms_per_step'])"
