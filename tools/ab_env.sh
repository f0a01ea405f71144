#!/usr/bin/env bash
# A/B of env-knob settings on the configs' bench steps (same binary, same box, interleaved reps).
# usage: SETS="base GSG_BWD_TFIRST=1 GSG_BWD_TFIRST=2,GSG_HEAD_DHFIRST=1" CFGS="2 3 4 5" TAG=x bash tools/ab_env.sh
O=gpurun_out/ab_${TAG:-x}
mkdir -p $O
for rep in ${REPS:-1 2}; do
  for set in $SETS; do
    envs=""; [ "$set" != base ] && envs=$(echo "$set" | tr ',' ' ')
    for c in ${CFGS:-2 3 4 5}; do
      env $envs python bench.py --config $c --no-cpu --no-e2e --steps ${STEPS:-30} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'set':'$set','rep':$rep,'cfg':$c,'ms':round(d['ms_per_step'],4),'p50':round(d['step_ms_dist']['p50'],4),'frac':round(d['roofline']['frac'],3)}))" >> $O/step.jsonl
    done
  done
done
