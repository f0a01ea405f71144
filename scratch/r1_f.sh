for c in none 0 10 25 50 100; do if [ $c = none ]; then unset GSG_SPMM_CARVEOUT; else export GSG_SPMM_CARVEOUT=$c; fi
WIDTHS=200,1024 timeout 300 python tools/spmm_bench.py 2>&1 | grep '^{' | sed "s/^/carve$c /"; done | tee gpurun_out/carve.jsonl
unset GSG_SPMM_CARVEOUT
timeout 600 ncu --set full --clock-control none -k regex:k_spmm_wide -s 2 -c 1 -f -o gpurun_out/spmm1024 env WIDTHS=1024 python tools/spmm_bench.py > gpurun_out/ncu_spmm.log 2>&1; echo ncu=$?
