# MT seq 256 tail size; LM gate multicast cluster size (final build, same box)
out=gpurun_out/${1:-r02_sweep2}; mkdir -p $out
for rep in 1 2; do
for t in 0 1500 2000 3000 5000; do
  MOE_FFN_DYN_TAIL=$t timeout 300 python bench.py --workload mt-l256 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/l256_t$t.json > $out/l256_t$t.log 2>&1
  python -c "import json;d=json.load(open('$out/l256_t$t.json'));print('mt-l256 dyn_tail $t','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done
for c in 4 2 1; do
  MOE_GATE_CLUSTER=$c timeout 300 python bench.py --workload lm --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/lm_c$c.json > $out/lm_c$c.log 2>&1
  python -c "import json;d=json.load(open('$out/lm_c$c.json'));print('lm gate cluster $c','ms',round(d['ms_per_step'],4),'gate us',round(d['stage_ms']['gate_topk']*1000,1))" >> $out/summary.txt 2>&1
done; done
cat $out/summary.txt
