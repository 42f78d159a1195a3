# cfg1 FFN forms after the size-gated H discard: 1-SM / CTA pairs x 128 / 256-token items
out=gpurun_out/${1:-r02_cfg1forms}; mkdir -p $out
for rep in 1 2; do
for v in "1sm 128 0" "pair 128 1" "1sm 256 0" "pair 256 1"; do
  set -- $v
  MOE_FFN_PAIR=$3 timeout 300 python bench.py --workload cfg1 --tile-n $2 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/$1_$2.json > $out/$1_$2.log 2>&1
  python -c "import json;d=json.load(open('$out/$1_$2.json'));print('$1 $2','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt
done; done
cat $out/summary.txt
