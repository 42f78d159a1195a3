# packed weights as 1-D bulk copies (MOE_FFN_BULK_W) vs tensor-map boxes
out=gpurun_out/${1:-r02_bulkw}; mkdir -p $out
for spec in "cfg1 X=1" "lm MOE_FFN_PAIR=0" "mt-l256 MOE_FFN_PAIR=0" "lm X=1"; do set -- $spec
for bw in 1 0 1 0; do
  env $2 MOE_FFN_BULK_W=$bw timeout 300 python bench.py --workload $1 --steps 30 --no-cpu-baseline --e2e-steps 3 --json-out $out/$1_$bw.json > $out/$1_$bw.log 2>&1
  python -c "import json;d=json.load(open('$out/$1_$bw.json'));print('$1 $2 bulk_w',$bw,'ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1),d['clocks']['sm_mhz'])" >> $out/summary.txt
done; done
cat $out/summary.txt
