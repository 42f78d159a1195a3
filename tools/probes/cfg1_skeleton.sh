# cfg1 FFN: per-CTA start/end spread (MOE_FFN_PROF) with and without work
# (MOE_FFN_DBG 31 = no loads, MMAs, TMEM loads or stores), plus the stage
# times of 1-SM 128 / 256-token items.
out=gpurun_out/${1:-r02_cfg1skel}; mkdir -p $out
for d in 0 31 21; do
  echo "dbg $d" >> $out/prof.txt
  MOE_FFN_DBG=$d MOE_FFN_PROF=1 timeout 300 python tools/prof_step.py --workload cfg1 --steps 3 2>&1 | grep "ffn prof" >> $out/prof.txt
done
for tn in 128 256; do
  timeout 300 python bench.py --workload cfg1 --tile-n $tn --steps 50 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/tn$tn.json > $out/tn$tn.log 2>&1
  python -c "import json;d=json.load(open('$out/tn$tn.json'));print('tile_n $tn','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1))" >> $out/prof.txt
done
cat $out/prof.txt
