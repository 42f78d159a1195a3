# FFN GEMM1->GEMM2 lag (items) sweep per workload (bench FFN stage + step)
for w in ${WS:-mt-l256}; do for lag in ${LAGS:-0 4 6 10 15 20}; do
  env $( [ $lag != 0 ] && echo MOE_FFN_LAG=$lag ) timeout 300 python bench.py --workload $w --steps 30 --no-cpu-baseline --e2e-steps 3 --no-clocks > /tmp/l.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/l.json').read().strip().splitlines()[-1]);print('$w lag',$lag,'ms',round(d['ms_per_step'],4),'ffn',round(d['stage_ms']['ffn_gemm1'],4))"
done; done
