L=paper_2303_06182_b200/libmoe_b200.so
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for w in lm mt cfg1; do echo "== $w"; bash tools/ab_bench.sh "$L@MOE_GATHER_TOKENS=0 $L@MOE_GATHER_TOKENS=1" 3 --workload $w; done
