#!/bin/bash
# FFN ablations on the LM shape: env knobs of the fused FFN, bench stage times.
#   MOE_FFN_DBG=1 skip B (activation) loads, 2 skip output stores
#   MOE_FFN_LAG   items between an item's GEMM1 and GEMM2 tiles
#   MOE_FFN_KCH=1 6 x 32 KB stages instead of 3 x 64 KB
out=${1:-gpurun_out/ffn_sweep.txt}
: > "$out"
run() {
  local tag="$1"; shift
  rm -f /tmp/b.json
  env "$@" timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 3 --json-out /tmp/b.json > /tmp/b.log 2>&1
  python - "$tag" >> "$out" <<'PY'
import json, os, sys
if not os.path.exists("/tmp/b.json"):
    print(f"{sys.argv[1]:28s} FAILED: " + open("/tmp/b.log").read()[-300:].replace("\n", " | "))
    sys.exit(0)
d = json.load(open("/tmp/b.json"))
print(f"{sys.argv[1]:28s} step {d['ms_per_step']:.4f} ms  ffn {d['stage_ms']['ffn_gemm1']*1e3:.1f} us  clocks {d['clocks']['sm_mhz'] if d.get('clocks') else None}")
PY
}
if [ -n "$SWEEP" ]; then for v in $SWEEP; do run "$v" $v; done; else
run base
run dbg1_noB MOE_FFN_DBG=1
run dbg2_nostore MOE_FFN_DBG=2
run dbg3 MOE_FFN_DBG=3
run kch1 MOE_FFN_KCH=1
for lag in 16 24 48 64; do run lag$lag MOE_FFN_LAG=$lag; done
run base_again
fi
cat "$out"
