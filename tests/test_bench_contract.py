"""bench.py contract on CPU: the reference arm (the reference's CPU path:
gating.cpp verbatim build + numpy/BLAS layer arithmetic) prints one JSON line
with the keys the driver reads, and exits 0 on every rank under torchrun."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _last_json(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


@pytest.mark.timeout(300)
def test_reference_arm_json_line():
    env = dict(os.environ, MOE_CPU_BASELINE_SECONDS="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1", "--steps", "1",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=280, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


@pytest.mark.timeout(300)
def test_reference_arm_under_torchrun_prints_once():
    env = dict(os.environ, MOE_CPU_BASELINE_SECONDS="2")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29571", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--workload", "cfg1", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=280, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"


@pytest.mark.timeout(200)
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_gpus_flag_relaunches_one_rank_per_gpu(scaling):
    """`bench.py --gpus 2` outside torchrun relaunches itself as 2 ranks (the
    form the driver may use); --dry-run stops before any GPU work."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--scaling", scaling],
                       cwd=ROOT, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 and d["n_gpus"] == 2 and d["scaling"] == scaling for d in lines)


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


@pytest.mark.gpu
@pytest.mark.timeout(400)
def test_b200_arm_json_line_on_gpu():
    """The driver's own arm on the B200 (short run): one JSON line with every
    key of the contract, the roofline / cpu_baseline / e2e / clocks objects,
    e2e copies counted, and a positive kernel-launch claim."""
    env = dict(os.environ, MOE_CPU_BASELINE_SECONDS="1", MOE_BENCH_CPU_DETAIL="0")
    r = subprocess.run([sys.executable, "bench.py", "--workload", "cfg1", "--steps", "5", "--warmup", "3",
                        "--e2e-steps", "4"], cwd=ROOT, capture_output=True, text=True, timeout=380, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    need = (KEYS - {"impl"}) | {"roofline", "clocks", "gpu_launches", "p50_ms"}
    assert need <= set(d), need - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    ro = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(ro) and ro["frac"] > 0
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 5 * 5
