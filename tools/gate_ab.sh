#!/bin/bash
# Gate A/B on one box: ncu launch list (cold, serialised) + MOE_GATE_PROF
# per-CTA phase times per workload, default vs MOE_GATE_SPLIT=0.
tag=${1:-gate_ab}
out=gpurun_out/$tag
mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
for w in ${WORKLOADS:-mt cfg1 lm}; do
  for v in default ${VARIANTS:-nosplit}; do
    env=""
    [ $v = nosplit ] && env="MOE_GATE_SPLIT=0"
    [ $v = pairoff ] && env="MOE_GATE_PAIR=0"
    env $env $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:gate -c 6 --csv \
      --log-file $out/launch_${w}_$v.csv python tools/prof_step.py --workload $w --steps 6 > /dev/null 2>&1
    env $env MOE_GATE_PROF=1 timeout 300 python tools/prof_step.py --workload $w --steps 4 > $out/prof_${w}_$v.log 2>&1
  done
done
for f in $out/launch_*.csv; do
  echo "$f $(python - "$f" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3}
v = [float(r[-1].replace(",", "")) * scale.get(r[-2], 1.0) for r in rows]
print(rows[0][4][:40] if rows else "", "grid", rows[0][8] if rows else "", "us:", ["%.1f" % x for x in v])
PY
)"
done > $out/summary.txt
grep -h "gate prof" $out/prof_*.log | tail -30 >> $out/summary.txt
cat $out/summary.txt
