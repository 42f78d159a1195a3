out=gpurun_out/r02_s8_cfg1sweep; mkdir -p $out
for rep in 1 2; do
for v in "X=0" "MOE_FFN_FENCE=0" "MOE_FFN_DISCARD=0" "MOE_FFN_FENCE=0 MOE_FFN_DISCARD=0"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 python bench.py --workload cfg1 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/$tag.json > $out/$tag.log 2>&1
  python -c "import json;d=json.load(open('$out/$tag.json'));print('$v','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt
done; done
cat $out/summary.txt
