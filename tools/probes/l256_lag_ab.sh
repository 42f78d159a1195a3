# MT seq 256: 4x lag for dynamic 256-token items (default now) vs the previous lag (MOE_FFN_LAG=15)
out=gpurun_out/${1:-r02_l256lag}; mkdir -p $out
for rep in 1 2 3 4; do
for v in new 15; do
  if [ $v = new ]; then unset MOE_FFN_LAG; else export MOE_FFN_LAG=$v; fi
  timeout 300 python bench.py --workload mt-l256 --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/l256_$v.json > $out/l256_$v.log 2>&1
  python -c "import json;d=json.load(open('$out/l256_$v.json'));print('mt-l256 lag $v','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done
unset MOE_FFN_LAG
timeout 600 python -m pytest tests -m gpu -q -k "parity or schedule or fused or ffn" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/summary.txt; tail -1 $out/pytest.log >> $out/summary.txt
cat $out/summary.txt
