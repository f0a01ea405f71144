timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_n.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_n.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_n.json 2>gpurun_out/bench_n.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_n.json'));print(d['ms_per_step'], d['value'], d['stages_ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_n.log 2>&1; echo ncu=$?
