#!/bin/bash
# GPU tests + the main bench lines (no ncu): a check after a kernel-side change.
tag=${1:-quick}; out=gpurun_out/$tag; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
for w in ${WORKLOADS:-lm mt mt-l256 cfg1}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --json-out $out/bench_$w.json > $out/bench_$w.log 2>&1
  echo "bench $w rc=$?" >> $out/status.txt
  python -c "import json;d=json.load(open('$out/bench_$w.json'));print('$w','ms',round(d['ms_per_step'],4),'ffn us',round(d['stage_ms']['ffn_gemm1']*1000,1),'e2e',d['e2e']['value'])" >> $out/status.txt 2>&1
done
tail -1 $out/pytest_gpu.log >> $out/status.txt
cat $out/status.txt
