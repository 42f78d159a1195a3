"""The C++ host path end to end: build/bin/moesim_measure drives the GPU layer
through include/moesim/gpu_layer.hpp (no CUDA runtime in the host program)
and writes the reference CLI's report schema (proj/tools/moesim.cpp:342-423)
with measured numbers."""
import csv
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "bin", "moesim_measure")


def _run(tmp_path, *args):
    out = tmp_path / "rep"
    r = subprocess.run([EXE, "--out", str(out), *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return out, r.stdout


def _summary(out):
    with open(out / "summary.csv") as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["metric", "value"]
    return {k: float(v) for k, v in rows[1:]}


def test_measure_report_schema_and_numerics(tmp_path):
    out, text = _run(tmp_path, "--experts", "16", "--topk", "2", "--tokens", "512", "--batches", "4",
                     "--token-dim", "256", "--hidden-dim", "512", "--mode", "both", "--capacity-factor", "0.5",
                     "--verify", "6")
    print(text)
    s = _summary(out)
    assert s["verify_rel_fro"] < 1e-2
    assert s["num_batches"] == 4 and s["total_tokens"] == 2048
    assert s["capacity"] == 256 and s["waste_factor"] == 4.0
    assert s["throughput_dynamic"] > 0 and s["throughput_static"] > 0
    with open(out / "latency.csv") as f:
        lat = list(csv.reader(f))
    assert lat[0] == ["component", "seconds"]
    names = [r[0] for r in lat[1:]]
    for mode in ("static", "dynamic"):
        for c in ("gate", "reorder", "a2a_size", "a2a_payload", "expert_compute", "cpu_gpu_transfer", "total"):
            assert f"{mode}.{c}" in names
    man = json.load(open(out / "manifest.json"))
    assert man["command"] == "measure" and "summary.csv" in man["outputs"]


def test_measure_with_expert_cache_and_gate(tmp_path):
    out, text = _run(tmp_path, "--experts", "16", "--topk", "2", "--tokens", "256", "--batches", "6",
                     "--token-dim", "256", "--hidden-dim", "256", "--mode", "dynamic", "--cache-size", "4",
                     "--active-frac", "0.5")
    with open(out / "cache.csv") as f:
        rows = list(csv.reader(f))
    assert rows[0][:4] == ["device", "accesses", "hits", "misses"]
    g = rows[-1]
    assert g[0] == "global" and int(g[1]) == int(g[2]) + int(g[3])
    out2, _ = _run(tmp_path, "--experts", "8", "--topk", "1", "--tokens", "300", "--batches", "2",
                   "--token-dim", "128", "--hidden-dim", "256", "--mode", "dynamic", "--gate", "--verify", "4")
    assert _summary(out2)["verify_rel_fro"] < 1e-2


def test_measure_replays_trace_file(tmp_path):
    """--trace: a JSON Lines routing trace (reference format) with batches of
    different lengths drives the GPU layer; --save-trace writes back the same
    bytes; the fp32 check uses the replayed routing."""
    rng = __import__("numpy").random.default_rng(3)
    E, k, lens = 12, 2, [200, 37, 256]
    lines = [json.dumps({"num_experts": E, "top_k": k, "version": 1}, separators=(",", ":"), sort_keys=True)]
    for b, n in enumerate(lens):
        toks = []
        for _ in range(n):
            e = rng.choice(E, size=k, replace=False).tolist()
            toks.append({"e": e, "w": [0.75, 0.25]})
        lines.append(json.dumps({"batch_id": b, "tokens": toks}, separators=(",", ":"), sort_keys=True))
    trace = tmp_path / "t.jsonl"
    trace.write_text("\n".join(lines) + "\n")
    saved = tmp_path / "saved.jsonl"
    out, text = _run(tmp_path, "--trace", str(trace), "--save-trace", str(saved), "--token-dim", "128",
                     "--hidden-dim", "256", "--mode", "dynamic", "--verify", "5")
    s = _summary(out)
    assert s["num_batches"] == 3
    assert s["verify_rel_fro"] < 1e-2
    assert saved.read_bytes() == trace.read_bytes()
    man = json.load(open(out / "manifest.json"))
    assert "file:" in json.dumps(man)
