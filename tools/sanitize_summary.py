"""Classify compute-sanitizer logs (tools/sanitize.sh):
  python tools/sanitize_summary.py <dir>
Per log: non-leak errors, leaks allocated by this library (libmoe*), leaks of
torch's caching allocator (freed by the process exit, not by the program),
and the tool's own summary line."""
import glob
import os
import re
import sys

d = sys.argv[1]
for f in sorted(glob.glob(os.path.join(d, "*.log"))):
    txt = open(f, errors="replace").read()
    blocks = re.split(r"^========= (?=\S)", txt, flags=re.M)
    errs, ours, torch_ = 0, 0, 0
    kinds = {}
    for b in blocks:
        head = b.split("\n", 1)[0]
        if head.startswith("Leaked"):
            if "libmoe" in b:
                ours += 1
            else:
                torch_ += 1
        elif head.startswith(("Invalid", "Error", "Program hit", "Out-of", "Misaligned", "Barrier",
                              "Uninitialized", "Race", "Warning")):
            errs += 1
            k = head[:60]
            kinds[k] = kinds.get(k, 0) + 1
    summ = [l for l in txt.splitlines() if "ERROR SUMMARY" in l or "RACECHECK SUMMARY" in l]
    ok = any(l.strip() == "OK" for l in txt.splitlines()) or ": 0 rows differ" in txt
    print(f"{os.path.basename(f):28s} errors={errs:<4d} lib_leaks={ours:<3d} torch_pool_leaks={torch_:<3d} "
          f"case_ok={ok!s:5s} {summ[-1].replace('=========', '').strip() if summ else ''}")
    for k, v in list(kinds.items())[:4]:
        print(f"    {v} x {k}")
