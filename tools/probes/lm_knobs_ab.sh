# LM step (graph replay, 200 steps) A/B of FFN fence form and the PDL trigger points, 3 alternating rounds
out=gpurun_out/${1:-r02_knobs}; mkdir -p $out
for rep in 1 2 3; do
for v in "BASE=1" "MOE_FFN_FENCE=0" "MOE_GATHER_LATE_TRIGGER=1" "MOE_COMBINE_LATE_TRIGGER=0" "MOE_ROUTE_LATE_TRIGGER=1" "MOE_FFN_LATE_TRIGGER=0"; do
  tag=$(echo $v | tr '=' '_')
  env $v timeout 300 python bench.py --workload lm --steps 200 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/$tag.json > $out/$tag.log 2>&1
  python -c "import json;d=json.load(open('$out/$tag.json'));print('$v','ms',round(d['ms_per_step'],4),'p50',round(d['p50_ms'],4))" >> $out/summary.txt 2>&1
done; done
cat $out/summary.txt
