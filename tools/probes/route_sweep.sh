#!/bin/bash
# ncu-timed route kernel for several per-block chunk sizes (units of 512 slots)
for c in 1 2 4 8; do
  MOE_ROUTE_CHUNK_UNITS=$c ncu --metrics gpu__time_duration.sum --clock-control none -k regex:route_kernel --csv \
    --log-file gpurun_out/route_sweep_$c.csv python tools/probes/route_bench.py > /dev/null 2>&1
  python3 - "$c" <<'PY'
import csv, sys
c = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/route_sweep_{c}.csv")))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]; iv = h.index("Metric Value")
vals = [float(r[iv]) for r in rows[start + 1:] if len(r) > iv]
# route_bench: 4 configs x 55 launches
for j, name in enumerate(["S2048E8", "S16384E512", "S6144E128", "S131072E512"]):
    seg = vals[j * 55 + 5:(j + 1) * 55]
    print(c, name, round(sum(seg) / len(seg) / 1000, 2), "us")
PY
done
