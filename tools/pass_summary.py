"""Copy one tools/round_pass.sh output directory into profiles/ and write its
summary (bench table, CPU baseline detail, cache line, ncu launch lists and
full-capture metrics).
  python tools/pass_summary.py gpurun_out/<tag> <prefix, e.g. r02_s3> "<title>"
"""
import json
import os
import shutil
import subprocess
import sys

src, prefix, title = sys.argv[1], sys.argv[2], sys.argv[3]
P = "profiles"


def ncu(kind, path):
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", kind, path], capture_output=True, text=True).stdout
    return out.split("\n", 2)[2] if out.count("\n") >= 2 else out


for f in ("launches_lm.csv", "launches_ep1.csv", "launches_mt.csv", "launches_mt-l256.csv", "launches_cfg1.csv"):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(P, f"{prefix}_ncu_{f}"))
rows = []
for w in ("lm", "mt", "mt_cpu", "mt-l256", "cfg1", "lm-static", "mt-static", "mt-cache_slots32"):
    f = os.path.join(src, f"bench_{w}.json")
    if not os.path.exists(f):
        continue
    shutil.copy(f, os.path.join(P, f"{prefix}_bench_{w}.json"))
    d = json.load(open(f))
    if "roofline" not in d:
        continue
    r, l, c = d["roofline"], d["layer_roofline"], d.get("clocks") or {}
    rows.append(f"| {w} | {d['ms_per_step']:.4f} | {d['value'] / 1e6:.3f} M | {d['e2e']['value'] / 1e6:.3f} M | "
                f"{r['frac']:.3f} ({r['bound']}) | {l['frac']:.3f} | {c.get('sm_mhz', 0):.0f} {c.get('reasons')} |")
for name, log in (("reference_lm", "bench_reference_lm.log"), ("ep2_onegpu_functional", "bench_ep2_onegpu.log")):
    p = os.path.join(src, log)
    if os.path.exists(p):
        lines = [x for x in open(p).read().splitlines() if x.startswith("{")]
        if lines:
            open(os.path.join(P, f"{prefix}_bench_{name}.json"), "w").write(lines[-1] + "\n")
pyt = open(os.path.join(src, "pytest_gpu.log")).read().strip().splitlines()[-1]
txt = [f"# {title}", "", f"`tools/round_pass.sh` on one B200.  GPU tests: `{pyt}`; `smoke()` ok.",
       "Bench lines: `" + prefix + "_bench_*.json`; ncu launch lists are the recipe's",
       "`--metrics gpu__time_duration.sum --clock-control none` pass (cold, serialised: compare",
       "SHARES of the step, not absolutes); the full capture is `--set full` of one step.", "",
       "| workload | ms / step | tokens/s | e2e tokens/s | FFN roofline frac | layer roofline frac | SM MHz, reasons |",
       "|---|---|---|---|---|---|---|"] + rows + [""]
mc = os.path.join(src, "bench_mt_cpu.json")
if os.path.exists(mc):
    c = json.load(open(mc)).get("cpu_baseline") or {}
    if c:
        txt += [f"CPU baseline (MT, {c['cores']} host cores): {c['value']:.0f} tokens/s full layer."]
        if "one_thread" in c:
            txt += [f"1-thread layer: {c['one_thread']['value']:.0f} tokens/s ({c['one_thread']['sample']})."]
        if "routing_1thread_s" in c:
            r = c["routing_1thread_s"]
            txt += [f"Reference routing alone, one thread, Batch prebuilt: dynamic_dispatch "
                    f"{r['dynamic_dispatch'] * 1e6:.1f} us, combine<float> {r['combine_dynamic'] * 1e6:.1f} us; "
                    f"GPU route stage {r['gpu_route_stage_s'] * 1e6:.1f} us.", ""]
ch = os.path.join(src, "bench_mt-cache_slots32.json")
if os.path.exists(ch):
    d = json.load(open(ch))
    k = d["cache"]
    txt += [f"Expert buffering (configs[4], {d['config']['cache_slots']} of {d['config']['E']} slots): "
            f"{d['ms_per_step']:.2f} ms/step, PCIe {k['h2d_gbs_achieved']:.1f} of {k['h2d_peak_gbs_measured']:.1f} GB/s "
            f"measured H2D peak ({k['pcie_frac']:.2f}); fully resident {d['fully_resident']['ms_per_step']:.3f} ms.", ""]
txt += ["## ncu launch list, LM step (single-GPU layer)", "", ncu("launches", os.path.join(src, "launches_lm.csv")),
        "## ncu launch list, LM step through the expert-parallel kernels at world 1", "",
        ncu("launches", os.path.join(src, "launches_ep1.csv")),
        ]
for w in ("mt", "mt-l256", "cfg1"):
    f = os.path.join(src, f"launches_{w}.csv")
    if os.path.exists(f):
        txt += [f"## ncu launch list, {w} step", "", ncu("launches", f)]
txt += ["## ncu --set full, LM step", "", ncu("full", os.path.join(src, "full_lm.ncu-rep")),
        "## ncu --set full, EP kernels at world 1", "", ncu("full", os.path.join(src, "full_ep1.ncu-rep"))]
open(os.path.join(P, f"{prefix}_ncu_summary.md"), "w").write("\n".join(txt).replace(src + "/", ""))
print("\n".join(txt[:20]))
