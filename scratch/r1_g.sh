timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k gemm > gpurun_out/pytest_g.log 2>&1; echo parity=$?; tail -3 gpurun_out/pytest_g.log
for t in 1 0; do for s in "20000,1024,200,0,0:relu" "20000,200,1024,0,1:mask" "20000,1024,1024,0,0:relu" "20000,1024,1024,0,1:mask" "8000,512,602,0,0:relu" "8000,602,512,0,1:mask" "12000,512,512,0,0:relu" "12000,300,512,0,1:mask"; do
  sh=${s%%:*}; ep=${s##*:}; GSG_GEMM_NO_TAIL=$t SHAPE=$sh EPI=$ep timeout 120 python tools/gemm_one.py | sed "s/^/notail=$t /"; done; done
