# cfg1 FFN schedule sweep: GEMM1 -> GEMM2 lag (items) x dynamically claimed tiles
# (MOE_FFN_DYN_TAIL: 0 = the last lag x MT2 tiles, 100000 = every tile)
out=gpurun_out/${1:-r02_cfg1sched}; mkdir -p $out
W=${W:-cfg1}
for rep in 1 2; do
for v in "0 0" "0 100000" "2 100000" "3 100000" "4 100000" "6 100000" "2 0" "4 0"; do
  set -- $v
  tag=lag$1_dyn$2
  MOE_FFN_LAG=$1 MOE_FFN_DYN_TAIL=$2 timeout 300 python bench.py --workload $W --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/$tag.json > $out/$tag.log 2>&1
  python -c "import json;d=json.load(open('$out/$tag.json'));print('$W lag $1 dyn $2','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done
cat $out/summary.txt
