#!/bin/bash
# Gate ablations (MOE_GATE_DBG) with per-CTA phase times (MOE_GATE_PROF):
# where the mainloop goes at each shape.  Wrong results by construction.
tag=${1:-gate_ablate}
out=gpurun_out/$tag
mkdir -p $out
for w in ${WORKLOADS:-lm mt cfg1}; do
  for d in ${DBGS:-0 1 2 3 4 8}; do
    MOE_GATE_DBG=$d MOE_GATE_PROF=1 timeout 300 python tools/prof_step.py --workload $w --steps 4 > $out/${w}_dbg$d.log 2>&1
    echo "$w dbg=$d $(grep -h 'gate prof' $out/${w}_dbg$d.log | tail -2 | tr '\n' ' ')" >> $out/summary.txt
  done
done
cat $out/summary.txt
