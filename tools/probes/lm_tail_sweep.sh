# LM / MT (CTA-pair FFN): size of the dynamically claimed tail (MOE_FFN_DYN_TAIL tiles; 0 = lag x MT2)
out=gpurun_out/${1:-r02_tail}; mkdir -p $out
for rep in 1 2; do
for W in lm mt; do
for t in 0 300 1000 3000 100000; do
  MOE_FFN_DYN_TAIL=$t timeout 300 python bench.py --workload $W --steps 100 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/${W}_t$t.json > $out/${W}_t$t.log 2>&1
  python -c "import json;d=json.load(open('$out/${W}_t$t.json'));print('$W dyn_tail $t','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done; done
cat $out/summary.txt
