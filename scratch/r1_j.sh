timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_j.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_j.log
for lib in old pred new; do cp scratch/libgsg_$lib.so paper_2010_03166_b200/libgsg.so
 for c in "5 200,1024" "4 200,1024" "3 300,512" "2 602,512"; do set -- $c; CFG=$1 WIDTHS=$2 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{' | sed "s/^/$lib /"; done; done | tee gpurun_out/prefetch_ab.jsonl
cp scratch/libgsg_new.so paper_2010_03166_b200/libgsg.so
for c in 5 4 3 2; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 30 > gpurun_out/bench_j$c.json 2>gpurun_out/bench_j$c.err; echo bench$c=$?
python -c "import json;d=json.load(open('gpurun_out/bench_j$c.json'));print($c, d['ms_per_step'], d['value'], d['stages_ms_per_step'])"; done
