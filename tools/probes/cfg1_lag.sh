# cfg1 FFN: GEMM1->GEMM2 lag (items) x FFN form
out=gpurun_out/${1:-r02_cfg1lag}; mkdir -p $out
for form in "128 -1" "256 1"; do set -- $form
for lag in 0 1 2 3 4 6; do
  env $( [ $lag != 0 ] && echo MOE_FFN_LAG=$lag ) $( [ $2 = 1 ] && echo MOE_FFN_PAIR=1 ) timeout 300 python bench.py --workload cfg1 --tile-n $1 --steps 30 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/t$1_l$lag.json > $out/t$1_l$lag.log 2>&1
  python -c "import json;d=json.load(open('$out/t$1_l$lag.json'));print('tile',$1,'lag',$lag,'ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt
done; done
cat $out/summary.txt
