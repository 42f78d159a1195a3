"""Per-source-line warp-stall samples of one kernel in an ncu report
(needs -lineinfo + --import-source on).
  python tools/ncu_lines.py <report.ncu-rep> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, fname = [], ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 6 and r[0].isdigit():
        try:
            out.append((int(r[4] or 0), fname, int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot = sum(o[0] for o in out)
print(f"total samples {tot}")
for s, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {f}:{ln}  {src[:100]}")
