out=gpurun_out/r02_cfg1ab; mkdir -p $out
for v in "128 -1" "128 1" "256 -1" "256 1"; do set -- $v
  for r in 1 2; do
  env $( [ $2 = 1 ] && echo MOE_FFN_PAIR=1 ) timeout 300 python bench.py --workload cfg1 --tile-n $1 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/t$1_p$2_$r.json > $out/t$1_p$2_$r.log 2>&1
  python -c "import json;d=json.load(open('$out/t$1_p$2_$r.json'));print('tile',$1,'pair',$2,'ms',round(d['ms_per_step'],4),{k:round(v*1000,1) for k,v in d['stage_ms'].items()}, d['roofline']['kernel'][:30])" >> $out/summary.txt
  done
done
cat $out/summary.txt
