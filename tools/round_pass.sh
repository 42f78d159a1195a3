#!/bin/bash
# One GPU call that refreshes every committed measurement: GPU tests, smoke,
# the bench line of every workload, the reference arm, the EP path (2 ranks
# sharing the one GPU: functional evidence only), ncu launch lists and full
# captures.  Outputs under gpurun_out/<tag>/.
tag=${1:-pass}
out=gpurun_out/$tag
mkdir -p $out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/status.txt
timeout 600 python bench.py --json-out $out/bench_lm.json > $out/bench_lm.log 2>&1; echo "bench lm rc=$?" >> $out/status.txt
for w in mt mt-l256 cfg1 lm-static mt-static; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --json-out $out/bench_$w.json > $out/bench_$w.log 2>&1
  echo "bench $w rc=$?" >> $out/status.txt
done
timeout 600 python bench.py --workload mt --json-out $out/bench_mt_cpu.json --steps 20 > $out/bench_mt_cpu.log 2>&1; echo "bench mt+cpu rc=$?" >> $out/status.txt
timeout 600 python bench.py --workload mt-cache --cache-slots 32 --json-out $out/bench_mt-cache_slots32.json > $out/bench_mt-cache.log 2>&1; echo "bench mt-cache rc=$?" >> $out/status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference_lm.log 2>&1; echo "reference rc=$?" >> $out/status.txt
MOE_BENCH_ONE_GPU_TEST=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > $out/bench_ep2_onegpu.log 2>&1; echo "ep2 one-gpu rc=$?" >> $out/status.txt
$NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/launches_lm.csv python tools/prof_step.py --steps 8 > /dev/null 2>&1; echo "ncu launches rc=$?" >> $out/status.txt
$NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/launches_ep1.csv python tools/prof_step.py --steps 8 --ep > /dev/null 2>&1
for w in mt mt-l256 cfg1; do
  $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/launches_$w.csv python tools/prof_step.py --workload $w --steps 8 > /dev/null 2>&1
done
$NCU --set full --clock-control none --import-source on -k regex:"gate_topk|route_kernel|gather|fused_ffn|combine" -s 5 -c 5 -o $out/full_lm python tools/prof_step.py --steps 3 > /dev/null 2>&1; echo "ncu full rc=$?" >> $out/status.txt
$NCU --set full --clock-control none --import-source on -k regex:"ep_" -s 5 -c 5 -o $out/full_ep1 python tools/prof_step.py --steps 3 --ep > /dev/null 2>&1
cat $out/status.txt
