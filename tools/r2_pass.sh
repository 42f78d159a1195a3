#!/bin/bash
# One GPU call: GPU tests, then the bench line of each workload with the
# per-stage breakdown, plus gate profiles (MOE_GATE_PROF) at MT / cfg1 / LM.
tag=${1:-pass}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
fi
for w in ${WORKLOADS:-lm mt mt-l256 cfg1 lm-static mt-static}; do
  timeout 400 python bench.py --workload $w --steps ${STEPS:-30} --no-cpu-baseline --json-out $out/bench_$w.json > $out/bench_$w.log 2>&1
  echo "bench $w rc=$?" >> $out/status.txt
done
for w in ${PROF_WORKLOADS:-mt cfg1 lm}; do
  MOE_GATE_PROF=1 timeout 300 python tools/prof_step.py --workload $w --steps 3 > $out/gateprof_$w.log 2>&1
done
cat $out/status.txt
