mkdir -p gpurun_out/sweep
for c in 1 2 3 4; do
  timeout 600 python bench.py --config $c --no-cpu --steps 50 > gpurun_out/sweep/c$c.json 2> gpurun_out/sweep/c$c.err; echo c$c=$?
done
timeout 600 python bench.py --config 1 --no-cpu --steps 50 --flush-l2 > gpurun_out/sweep/c1_flush.json 2> gpurun_out/sweep/c1_flush.err; echo c1f=$?
timeout 600 python bench.py --config 1 --no-cpu --steps 50 --batch 64 > gpurun_out/sweep/c1_b64.json 2> gpurun_out/sweep/c1_b64.err; echo c1b=$?
timeout 600 python bench.py --config 5 --no-cpu --steps 30 --pool 8 --no-e2e > gpurun_out/sweep/c5_pool8.json 2> gpurun_out/sweep/c5_pool8.err; echo c5p8=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01d.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
for s in "20000,1024,200,0,0:relu" "20000,200,1024,0,1:mask" "20000,107,1024,0,0:relu" "20000,1024,1024,0,0:relu"; do
  sh=${s%%:*}; ep=${s##*:}; tag=$(echo $sh | tr ',' '_')
  SHAPE=$sh EPI=$ep timeout 120 python tools/gemm_one.py
  SHAPE=$sh EPI=$ep ITERS=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -f -o gpurun_out/gemm_$tag env GRAPH=0 python tools/gemm_one.py > gpurun_out/ncu_gemm_$tag.log 2>&1; echo ncu_$tag=$?
done
