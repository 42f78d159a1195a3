# new pair-kernel tail default (>= 7 waves of pair-tiles) vs the old one (the
# GEMM2-only segment: MOE_FFN_DYN_TAIL=240 -> 120 pair-tiles), same box
out=gpurun_out/${1:-r02_tailab}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/summary.txt; tail -1 $out/pytest.log >> $out/summary.txt
for rep in 1 2 3; do
for W in lm mt mt-l256 lm-static; do
for t in new 240; do
  if [ $t = new ]; then unset MOE_FFN_DYN_TAIL; else export MOE_FFN_DYN_TAIL=$t; fi
  timeout 300 python bench.py --workload $W --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/${W}_$t.json > $out/${W}_$t.log 2>&1
  python -c "import json;d=json.load(open('$out/${W}_$t.json'));print('$W tail $t','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt 2>&1
done; done; done
unset MOE_FFN_DYN_TAIL
cat $out/summary.txt
