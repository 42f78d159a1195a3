# cfg1: 1-SM kernel at 256-token items with one 256-row token box per k chunk
# (MOE_FFN_ROWS256=1) vs four 64-row boxes (0), against the default 128-token items
out=gpurun_out/${1:-r02_rows256}; mkdir -p $out
for rep in 1 2 3; do
for v in "128 1" "256 1" "256 0"; do
  set -- $v
  MOE_FFN_PAIR=0 MOE_FFN_ROWS256=$2 timeout 300 python bench.py --workload cfg1 --tile-n $1 --steps 100 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/t$1_r$2.json > $out/t$1_r$2.log 2>&1
  python -c "import json;d=json.load(open('$out/t$1_r$2.json'));print('tile_n $1 rows256 $2','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "ffn or fused or parity" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/summary.txt; tail -1 $out/pytest.log >> $out/summary.txt
cat $out/summary.txt
