# LM (CTA-pair FFN): GEMM1 -> GEMM2 lag (items) sweep on the final build
out=gpurun_out/${1:-r02_lmlag}; mkdir -p $out
W=${W:-lm}
for rep in 1 2; do
for lag in 0 15 22 40 60; do
  MOE_FFN_LAG=$lag timeout 300 python bench.py --workload $W --steps 100 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/${W}_lag$lag.json > $out/${W}_lag$lag.log 2>&1
  python -c "import json;d=json.load(open('$out/${W}_lag$lag.json'));print('$W lag $lag','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done
cat $out/summary.txt
