# cfg1 FFN ablations (MOE_FFN_DBG, 1-SM kernel) + per-CTA spread (MOE_FFN_PROF)
out=gpurun_out/${1:-r02_ffnabl}; mkdir -p $out
for d in ${DBGS:-0 1 2 4 8 16 17 20 21 29 31} ; do
  MOE_FFN_DBG=$d timeout 300 python bench.py --workload ${W:-cfg1} --steps 30 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/d$d.json > $out/d$d.log 2>&1
  python -c "import json;d=json.load(open('$out/d$d.json'));print('dbg',$d,'ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/summary.txt
done
MOE_FFN_PROF=1 timeout 300 python tools/prof_step.py --workload ${W:-cfg1} --steps 3 > $out/prof.log 2>&1
MOE_FFN_PAIR=1 MOE_FFN_PROF=1 timeout 300 python tools/prof_step.py --workload ${W:-cfg1} --tile-n 256 --steps 3 > $out/prof_pair256.log 2>&1
cat $out/summary.txt; grep -h "prof\|ffn" $out/prof.log $out/prof_pair256.log | tail -6
