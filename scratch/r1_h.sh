for cfg in "GSG_GEMM_NO_TAIL=1" "GSG_TAIL_S=2" "GSG_TAIL_S=3" "GSG_TAIL_S=3 GSG_TAIL_NORED=1" "GSG_TAIL_S=2 GSG_TAIL_NORED=1"; do
 for s in "20000,1024,1024,0,0:relu" "20000,200,1024,0,1:mask"; do sh=${s%%:*}; ep=${s##*:};
  env $cfg SHAPE=$sh EPI=$ep ITERS=50 timeout 120 python tools/gemm_one.py | sed "s/^/$cfg /"; done; done
