#!/usr/bin/env bash
# A/B of an env knob on the SpMM widths and the configs' steps (same binary, same box, interleaved).
# usage: KNOB=GSG_SPMM_DYN VALS="0 1" TAG=x bash tools/ab_dyn.sh
O=gpurun_out/ab_${TAG:-x}
mkdir -p $O
for rep in 1 2; do
  for v in $VALS; do
    for c in 2 3 4 5; do
      env $KNOB=$v CFG=$c WIDTHS=${WIDTHS:-200,512,1024} python tools/spmm_bench.py 2>/dev/null | sed "s/^/{\"v\": \"$v\", \"rep\": $rep, \"row\": /; s/\$/}/" >> $O/spmm.jsonl
    done
  done
  for v in $VALS; do
    for c in 2 3 4 5; do
      env $KNOB=$v python bench.py --config $c --no-cpu --no-e2e --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'v':'$v','rep':$rep,'cfg':$c,'ms':d['ms_per_step'],'frac':d['roofline']['frac']}))" >> $O/step.jsonl
    done
  done
done
