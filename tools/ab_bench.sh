#!/bin/bash
# A/B of two builds of libmoe_b200.so on the same box: alternates runs of
# bench.py with MOE_LIB_PATH=<lib A> and <lib B>, prints ms/step and FFN ms.
#   tools/ab_bench.sh build/ab/libmoe_b200_base.so paper_2303_06182_b200/libmoe_b200.so [rounds] [bench args]
A=$1; B=$2; R=${3:-3}; shift 3
for i in $(seq 1 $R); do
  for lib in "$A" "$B"; do
    MOE_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-clocks "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$lib" <<'PY'
import json, os, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    st = d.get("stage_ms", {})
    print(f"{os.path.basename(sys.argv[1]):28s} step {d['ms_per_step']:.4f} ms  ffn {st.get('ffn_gemm1', 0) + st.get('ffn_gemm2', 0):.4f} ms  "
          f"gate {st.get('gate_topk', 0)*1e3:.1f} route {st.get('route', 0)*1e3:.1f} gather {st.get('gather', 0)*1e3:.1f} "
          f"combine {st.get('combine', 0)*1e3:.1f} us")
except Exception as e:
    print(sys.argv[1], "failed:", e, open("gpurun_out/ab.err").read()[-500:])
PY
  done
done
