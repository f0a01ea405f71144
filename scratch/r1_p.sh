for nt in 0 1; do for s in "20000,1024,200,0,0:relu" "20000,200,1024,0,1:mask" "20000,107,1024,0,0:relu" "20000,1024,107,0,1:mask" "20000,1024,1024,0,0:relu" "20000,1024,1024,0,1:mask" "8000,512,602,0,0:relu" "8000,602,512,0,1:mask" "12000,512,512,0,0:relu" "12000,300,512,0,1:mask" "16000,1024,1024,0,0:relu"; do
  sh=${s%%:*}; ep=${s##*:}; GSG_GEMM_NO_TMA_STORE=$nt SHAPE=$sh EPI=$ep ITERS=20 timeout 120 python tools/gemm_one.py | sed "s/^/notma=$nt /"; done; done
for s in "16000,1024,1024,0,0:relu" "16000,1024,200,0,0:relu" "16000,200,1024,0,1:mask"; do sh=${s%%:*}; ep=${s##*:}; PREC=bf16 SHAPE=$sh EPI=$ep ITERS=20 timeout 120 python tools/gemm_one.py; done
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.json 2>&1; echo gb=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config 2 --steps 2 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo ncu2=$?
