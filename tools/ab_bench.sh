#!/bin/bash
# Same-box A/B of several builds of libmoe_b200.so: alternates bench.py runs
# with MOE_LIB_PATH=<lib>, prints ms/step and per-stage times.
#   tools/ab_bench.sh "libA.so libB.so [...]" [rounds] [bench args]
# Env knobs for a variant: "libB.so@A=1,B=2" runs libB with those env vars.
LIBS=$1; R=${2:-3}; shift 2
for i in $(seq 1 $R); do
  for spec in $LIBS; do
    lib=${spec%%@*}; envs=""
    [ "$spec" != "$lib" ] && envs=${spec#*@} && envs=${envs//,/ }
    env $envs MOE_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-clocks "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err
    python - "$spec" <<'PY'
import json, os, sys
try:
    d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
    st = d.get("stage_ms", {})
    print(f"{os.path.basename(sys.argv[1]):36s} step {d['ms_per_step']:.4f} ms  ffn {st.get('ffn_gemm1', 0) + st.get('ffn_gemm2', 0):.4f} ms  "
          f"gate {st.get('gate_topk', 0)*1e3:.1f} route {st.get('route', 0)*1e3:.1f} gather {st.get('gather', 0)*1e3:.1f} "
          f"combine {st.get('combine', 0)*1e3:.1f} us  e2e {d['e2e']['ms_per_step']:.4f} ms", flush=True)
except Exception as e:
    print(sys.argv[1], "failed:", e, open("gpurun_out/ab.err").read()[-500:])
PY
  done
done
