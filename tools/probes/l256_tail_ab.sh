# MT seq 256 (256-token items): dynamically claimed tail 0 (default) vs larger, 3 rounds
out=gpurun_out/${1:-r02_l256tail}; mkdir -p $out
for rep in 1 2 3; do
for t in 0 5000 10000; do
  MOE_FFN_DYN_TAIL=$t timeout 300 python bench.py --workload mt-l256 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/l256_t$t.json > $out/l256_t$t.log 2>&1
  python -c "import json;d=json.load(open('$out/l256_t$t.json'));print('mt-l256 dyn_tail $t','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done
for t in 0 5000; do
  MOE_FFN_DYN_TAIL=$t timeout 300 python bench.py --workload mt-static --steps 10 --no-cpu-baseline --no-clocks --e2e-steps 2 --json-out $out/mts_t$t.json > $out/mts_t$t.log 2>&1
  python -c "import json;d=json.load(open('$out/mts_t$t.json'));print('mt-static dyn_tail $t','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done
cat $out/summary.txt
