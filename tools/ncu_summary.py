"""Summarise ncu captures into committed text under profiles/.

  python tools/ncu_summary.py launches <launches.csv>           -> per-kernel launch table
  python tools/ncu_summary.py full <report.ncu-rep> [...]       -> key metrics per kernel launch
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%elapsed"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct", "stall_long_sb_%"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    order = []
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
        if name not in agg:
            order.append(name)
        v = float(r[iv].replace(",", ""))
        agg[name].append(v / 1000.0 if r[iu] == "ns" else v)
    SETUP = ("fill_uniform", "pack_tiles")  # one-time data / weight setup, not part of a step
    tot = sum(sum(v) for n, v in agg.items() if not any(x in n for x in SETUP))
    out = ["| kernel | launches | mean us | min us | max us | share of step |", "|---|---|---|---|---|---|"]
    for n in order:
        v = agg[n]
        share = "" if any(x in n for x in SETUP) else f"{100 * sum(v) / tot:.1f}%"
        out.append(f"| `{n}` | {len(v)} | {sum(v) / len(v):.1f} | {min(v):.1f} | {max(v):.1f} | {share} |")
    return "\n".join(out)


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
        parts = []
        seen = set()
        for key, label in KEYS:
            cols = [j for j, n in enumerate(h) if n == key or n.endswith("." + key)]
            if cols and label not in seen:
                i = cols[0]
                seen.add(label)
                parts.append(f"{label}={r[i]} {units[i]}".strip())
        out.append(f"- `{name}`: " + "; ".join(parts))
    return "\n".join(out)


if __name__ == "__main__":
    mode = sys.argv[1]
    for p in sys.argv[2:]:
        print(f"### {p}\n")
        print(launches(p) if mode == "launches" else full(p))
        print()
