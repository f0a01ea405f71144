timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
for c in 5 2 3; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 30 > gpurun_out/bench_q$c.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_q$c.json'));print($c, d['ms_per_step'], d['stages_ms_per_step'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2q.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu2=$?
