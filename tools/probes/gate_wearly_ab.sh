# Gate: Wg boxes issued before griddepcontrol.wait (MOE_GATE_W_EARLY=1, default) vs after
out=gpurun_out/${1:-r02_wearly}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -k "gate or parity or layer" > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/summary.txt; tail -1 $out/pytest.log >> $out/summary.txt
for rep in 1 2 3; do
for w in lm mt cfg1; do
for v in 1 0; do
  MOE_GATE_W_EARLY=$v timeout 300 python bench.py --workload $w --steps 100 --no-cpu-baseline --no-clocks --e2e-steps 3 --json-out $out/${w}_$v.json > $out/${w}_$v.log 2>&1
  python -c "import json;d=json.load(open('$out/${w}_$v.json'));print('$w w_early=$v','ms',round(d['ms_per_step'],4),'gate us',round(d['stage_ms']['gate_topk']*1000,1))" >> $out/summary.txt 2>&1
done; done; done
for v in 1 0; do
  MOE_GATE_W_EARLY=$v /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gate -c 40 --csv python tools/prof_step.py --steps 8 2>/dev/null | grep -c gate_topk >> $out/summary.txt
done
cat $out/summary.txt
