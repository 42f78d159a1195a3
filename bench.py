#!/usr/bin/env python
"""bench.py -- MoE-layer tokens/s & p50 latency, dynamic gating, on B200.

Metric (BASELINE.json): "MoE-layer tokens/s & p50 latency, dynamic gating,
1/2/4/8 B200 vs CPU ref".  Workload at N=1: configs[1], the LM MoE layer
(TD=1024, HD=4096, E=512, top-2, batch 8 x seq 2048 = 16384 tokens), dynamic
gating, bf16 weights/activations with fp32 accumulation, random-init experts,
synthetic tokens.

A step = one MoE-layer forward (gate + top-k, dispatch, gather, grouped expert
FFN, combine) over one batch of tokens resident in HBM.  Timing: W warm-up
steps, then K steps bracketed by barrier + cuda synchronize, CUDA events on the
launching stream, max over ranks.  The per-step working set (8.7 GB of expert
weights) is ~70x the 126 MB L2, so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload lm|mt|mt-l256|cfg1|lm-static|mt-static|mt-cache]

N > 1 (torchrun): one rank per GPU, expert parallelism -- E/N experts per GPU
(greedy load-balanced placement), 16384 tokens per GPU (weak scaling), NCCL
count exchange + variable all-to-all over NVLink (--replicas: full copies).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (S, TD, HD, E, k, mode, C, description)
    "lm": (16384, 1024, 4096, 512, 2, "dynamic", 0.0,
           "configs[1]: LM MoE layer TD=1024 HD=4096 E=512 top-2, batch 8 x seq 2048, dynamic gating"),
    "lm-static": (16384, 1024, 4096, 512, 2, "static", 0.05,
                  "configs[1] comparison: LM layer, static gating CF=0.05 (cap 820)"),
    "mt": (6144, 2048, 8192, 128, 2, "dynamic", 0.0,
           "configs[2]: MT MoE layer TD=2048 HD=8192 E=128 top-2, batch 48 x seq 128, dynamic gating"),
    "mt-l256": (12288, 2048, 8192, 128, 2, "dynamic", 0.0,
                "configs[2], longer sequences: MT MoE layer TD=2048 HD=8192 E=128 top-2, batch 48 x seq 256, "
                "dynamic gating (SURVEY.md section 8 cfg3 'also report L=256')"),
    "mt-static": (6144, 2048, 8192, 128, 2, "static", 1.0,
                  "configs[2] comparison: MT layer, static gating CF=1 (cap 6144)"),
    "cfg1": (2048, 1024, 4096, 8, 1, "dynamic", 0.0,
             "configs[0] shape: LM layer TD=1024 HD=4096 E=8 top-1, 2048 tokens"),
    "mt-cache": (48, 2048, 8192, 128, 2, "dynamic", 0.0,
                 "configs[4]: MT layer E=128 top-2 with expert buffering (LIFO GPU cache over pinned host "
                 "experts), decoder step batch 48, skewed routing zipf 1.2 / persist 0.9 / active 0.75"),
}
STAGES = ["gate_topk", "route", "gather", "ffn_gemm1", "ffn_gemm2", "combine"]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def cpu_seconds() -> float:
    """Timed CPU work per CPU-baseline measurement (>= 10 s by default;
    MOE_CPU_BASELINE_SECONDS shortens it for the CPU contract tests)."""
    return float(os.environ.get("MOE_CPU_BASELINE_SECONDS", "10"))


def sustained_tflops(default):
    """bf16 TF/s sustained under the power cap (for a kernel timed inside a
    long step, B200_PROFILING.md); the burst figure if absent."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f).get("bf16_tflops_sustained", default))
    except Exception:
        return 1400.0 if default == 1590.0 else default


class ClockSampler:
    """nvidia-smi clocks/throttle sampler (runs across the timed region)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t_start = self.t_stop = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 5:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def mark_start(self):
        self.t_start = time.time()

    def mark_stop(self):
        self.t_stop = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        inside = [r for (t, r) in self.rows if self.t_start and self.t_start - 0.06 <= t <= (self.t_stop or t) + 0.06]
        use = inside or [r for (_, r) in self.rows[-3:]]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in use:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[2]))
                mx.append(float(f[3]))
            except Exception:
                continue
            for n, v in zip(names, f[6:10]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(use), "samples_in_timed_region": len(inside)}


def ffn_bytes(rows, active, TD, HD, one_launch):
    """Algorithmic HBM bytes of the grouped FFN, bf16: each active expert's W1
    and W2 read once, Xp read, Yw written; the two-launch form also writes H
    and reads it back (the fused launch keeps H in L2)."""
    h = 0 if one_launch else 2 * rows * HD * 2
    return active * 2 * HD * TD * 2 + rows * TD * 2 + rows * TD * 2 + h


# Read-only HBM ceiling measured on B200 for the FFN's weight-stream pattern
# (1-D bulk TMA into 148 SMs, profiles/r01_s2_hbm_read_ceiling.txt): the copy
# peak in MEASURED_PEAKS counts reads + writes, so a read stream can exceed it.
READ_CEILING_GBS = 7430.0


def layer_roofline(S, TD, HD, E, k, active, hbm_gbs, tflops):
    """F = 2 S TD E + 4 k S TD HD; B = S TD 2 + E TD 2 +
    A 2 TD HD 2 + S TD 2 (bf16).  T_roof = max(F / P_tc, B / BW)."""
    F = 2.0 * S * TD * E + 4.0 * k * S * TD * HD
    B = S * TD * 2 + E * TD * 2 + active * 2 * TD * HD * 2 + S * TD * 2
    return max(F / (tflops * 1e12), B / (hbm_gbs * 1e9)), F, B


def load_traffic(workload):
    """dram bytes per FFN launch pair from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ffn_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


def _write_line(text):
    """One line to stdout in as few write(2) calls as the pipe allows: under
    torchrun every rank shares the parent's stdout, and print() may split a
    line around another rank's output."""
    sys.stdout.flush()
    buf = (text + "\n").encode()
    while buf:
        buf = buf[os.write(1, buf):]


def emit(line, args):
    """The one JSON line on stdout (+ --json-out copy)."""
    _write_line(json.dumps(line))
    if getattr(args, "json_out", None):
        with open(args.json_out, "w") as f:
            json.dump(line, f, indent=1)


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only knob: run N ranks on one GPU over gloo (exercises the EP code
    # path on a single-GPU box; the numbers are not a measurement)
    if os.environ.get("MOE_BENCH_ONE_GPU_TEST") == "1":
        local = 0
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("MOE_BENCH_ONE_GPU_TEST") != "1" and torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} GPU(s) visible")
        torch.cuda.set_device(local)
        if os.environ.get("MOE_BENCH_ONE_GPU_TEST") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def run_reference(args):
    """--impl reference: the reference's CPU path for this layer on the host
    cores (oracle/cpu_layer.py; routing = the reference's gating.cpp compiled
    verbatim), each step a bounded sample of the same workload."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.cpu_layer import CpuLayer, cpu_layer_bench

    S, TD, HD, E, k, mode, C, desc = WORKLOADS[args.workload]
    L = CpuLayer(S, TD, HD, E, k)
    warm = max(0, min(args.warmup, 3))  # full layer passes (~2.6 s each at LM)
    for _ in range(warm):
        L.run()
    # each step: full layer passes until >= 10 s of CPU work, median pass
    vals, secs = [], []
    r = None
    for _ in range(max(1, min(args.steps, 3))):
        r = cpu_layer_bench(S, TD, HD, E, k, min_seconds=cpu_seconds(), layer=L)
        vals.append(r["tokens_per_s"])
        secs.append(r["seconds_per_layer"])
    vals.sort()
    v = vals[len(vals) // 2]
    secs.sort()
    sample = r["sample"]
    line = {
        "metric": "MoE-layer tokens/s (dynamic gating)", "value": v, "unit": "tokens/s",
        "impl": "reference", "n_gpus": world, "steps": len(vals), "warmup": warm,
        "ms_per_step": secs[len(secs) // 2] * 1e3, "p50_ms": secs[len(secs) // 2] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter-hash uniform tokens; random-init experts)",
        "config": {"workload": desc, "S": S, "TD": TD, "HD": HD, "E": E, "top_k": k, "gating": mode},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "port",
                         "sample": sample, "cpu_model": r["cpu_model"], "host_cpus": r["host_cpus"]},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "breakdown_s": r["breakdown_s"],
    }
    emit(line, args)


def run_ep(args, world, rank, local):
    """N > 1: expert parallelism.  E/N experts per GPU (placement: the
    reference's greedy policy -- the C++ host library's greedy_place -- on a
    calibration routing histogram, or contiguous).  --scaling weak: S tokens
    per GPU; strong: the S tokens of one batch split over the GPUs, token t on
    GPU t % N (exchange.cpp:35-37).  Exchange (--ep-transport), both in the C
    ABI (moe_ep_*):
      p2p   (default) the layer's own kernels over NVLink peer memory:
            counts published into every peer's window, token rows gathered
            straight into the owner's receive buffer, outputs read back by the
            combine -- no host sync, the step is one CUDA graph
      nccl  NCCL count all-gather + host sync + grouped ncclSend/ncclRecv of
            the rows and back (csrc/ep_nccl.cu), the comparison path"""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2303_06182_b200 import placement as PL
    from paper_2303_06182_b200.ep import PeerExpertParallelMoE, Placement
    from paper_2303_06182_b200.layer import Context, LayerShape, make_tokens, make_weights

    S_job, TD, HD, E, k, mode, C, desc = WORKLOADS[args.workload]
    if mode != "dynamic":
        raise SystemExit("expert parallelism is implemented for dynamic gating")
    hbm_gbs, tflops, peak_kind = measured_peaks()
    ctx = Context.get(local)
    shape = LayerShape(TD, HD, E, k)
    Wg, W1, W2 = make_weights(shape, seed=2303061820, ctx=ctx)
    strong = args.scaling == "strong"
    if strong:
        # one global batch; this rank holds tokens t = rank, rank + N, ...
        xg = make_tokens(S_job, TD, seed=2303061820, ctx=ctx)
        x = xg[rank::world].contiguous()
        del xg
        S = x.shape[0]
        S_total = S_job
        S_max = (S_job + world - 1) // world
    else:
        x = make_tokens(S_job, TD, seed=2303061820 + rank, ctx=ctx)
        S = S_job
        S_max = S_job
        S_total = S_job * world
    # calibration history for the placement: one gate pass over a DIFFERENT
    # batch (the two-half protocol of the reference CLI, tools/moesim.cpp:
    # 451-492: place on one half of the trace, run on the other)
    import ctypes

    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    cur = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def expert_hist(tokens):
        n = tokens.shape[0]
        idx = torch.empty(n, k, dtype=torch.int32, device="cuda")
        w = torch.empty(n, k, dtype=torch.float32, device="cuda")
        ctx.lib.moe_gate_topk(ctx.h, P(tokens), P(Wg), n, TD, E, k, P(idx), P(w), None, cur)
        h = torch.bincount(idx.view(-1).long(), minlength=E).double()
        dist.all_reduce(h)
        return h.cpu().numpy()

    x_cal = make_tokens(S, TD, seed=2303061820 + 7919 + rank, ctx=ctx)
    hist = expert_hist(x_cal)[:, None] / (S * k * world)
    del x_cal
    hist_run = expert_hist(x)[:, None] / (S * k * world)
    if args.placement == "greedy":
        pl = Placement.greedy(hist, world)
    else:
        pl = Placement.contiguous(E, world)
    contig = PL.contiguous_place(E, world)
    balance = {
        "placement": args.placement, "history": "gate routing of a separate calibration batch",
        "ideal_load": 1.0 / world,
        "max_load_calibration": pl.balance(hist)["max_load"],
        "max_load_run_batch": pl.balance(hist_run)["max_load"],
        "contiguous_max_load_run_batch": PL.eval_balance(contig, world, hist_run)["max_load"],
    }
    loc = torch.from_numpy(pl.local_experts(rank)).long().cuda()
    W1l, W2l = W1[loc].contiguous(), W2[loc].contiguous()
    del W1, W2
    torch.cuda.empty_cache()
    p2p = args.ep_transport == "p2p"
    transport_note = ""
    layer = None
    if p2p:
        from paper_2303_06182_b200.ep import PeerMemoryUnavailable

        try:
            layer = PeerExpertParallelMoE(ctx, pl, shape, Wg, W1l, W2l, S_max, rank)
        except PeerMemoryUnavailable as e:  # raised on every rank: fall back together
            p2p = False
            transport_note = f"p2p unavailable ({e}); NCCL fallback"
    if layer is None:
        layer = PeerExpertParallelMoE(ctx, pl, shape, Wg, W1l, W2l, S_max, rank, transport="nccl")
    use_graph = p2p and not args.no_graph  # NCCL forwards have a host sync: eager
    fwd = lambda xx, st, out=None: layer.forward(xx, st, out=out, graph=use_graph)  # noqa: E731
    check = layer.check_errors
    # p2p: gate, route, publish, dispatch, recv, FFN, done, combine;
    # nccl: gate, route, gather, regroup, recv, FFN, regroup, combine (+ NCCL's own)
    n_launch = 8
    del W1l, W2l  # the EP layer keeps its tile-packed copy
    torch.cuda.empty_cache()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
    out_buf = torch.empty_like(x)
    K, W = args.steps, args.warmup
    with torch.cuda.stream(stream):
        for _ in range(W):
            out = fwd(x, stream, out_buf)
    stream.synchronize()
    check(stream)
    sampler = ClockSampler(local) if not args.no_clocks else None
    if sampler:
        sampler.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark_start()
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(K):
            step_ev[i].record(stream)
            out = fwd(x, stream, out_buf)
        step_ev[K].record(stream)
        ev1.record(stream)
    stream.synchronize()
    if sampler:
        sampler.mark_stop()
    barrier(world)
    elapsed = max_over_ranks(ev0.elapsed_time(ev1), world)
    steps = [step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(K)]
    p50 = max_over_ranks(float(np.median(steps)), world)
    p90 = max_over_ranks(float(np.percentile(steps, 90)), world)
    if sampler:
        sampler.stop()
    check(stream)
    v = layer.view(S)
    cnt = v["counts"].cpu().numpy().reshape(world, E // world).sum(1)
    recv_rows = v["recv_rows"]
    sent_off = int(cnt.sum() - cnt[rank])
    # measured per-GPU load: rows each GPU's experts received this step
    rr = torch.tensor([recv_rows], dtype=torch.int64, device="cuda")
    all_rr = [torch.zeros_like(rr) for _ in range(world)]
    dist.all_gather(all_rr, rr)
    rows_per_gpu = [int(t.item()) for t in all_rr]
    balance["measured_rows_per_gpu"] = rows_per_gpu
    balance["measured_max_load"] = max(rows_per_gpu) / max(sum(rows_per_gpu), 1)
    balance["measured_max_over_mean"] = max(rows_per_gpu) / max(np.mean(rows_per_gpu), 1e-9)
    # per-stage events from a separate untimed pass of eager forwards
    # (collective: every rank runs it); median per stage, max over ranks
    layer.enable_timing(True)
    per = []
    with torch.cuda.stream(stream):
        for _ in range(5):
            layer.forward(x, stream, out=out_buf, graph=False)
            per.append(layer.stage_times())
    layer.enable_timing(False)
    ep_stage = {kk: max_over_ranks(float(np.median([p_[kk] for p_ in per])), world) for kk in per[0]}
    # e2e: pinned host tokens in, host output out, copies inside the timed region
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    xd = torch.empty_like(x)
    od = torch.empty_like(x)
    Ke = max(3, min(K, args.e2e_steps))
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(Ke):
            xd.copy_(xh, non_blocking=True)
            o = fwd(xd, stream, od)
            oh.copy_(o, non_blocking=True)
        e1.record(stream)
    stream.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / Ke, world)
    check(stream)
    if rank != 0:
        layer.close()
        return
    ms = elapsed / K
    El = E // world
    wbytes = El * 2 * TD * HD * 2
    achieved = wbytes / (ms * 1e-3) / 1e9
    xbytes = 2 * sent_off * TD * 2  # token rows out + expert outputs back, off-GPU
    transport = ("NVLink peer memory: count publish + gather fused with the payload all-to-all + "
                 "return fused with the combine, one CUDA graph per step" if p2p else
                 "NCCL (C ABI): count all-gather + host sync + grouped send/recv of the rows and back")
    line = {
        "metric": "MoE-layer tokens/s (dynamic gating)", "value": S_total / (ms * 1e-3), "unit": "tokens/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms, "p50_ms": p50, "p90_ms": p90,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-hash uniform tokens; random-init experts, std 1/sqrt(fan-in))",
        "config": {"workload": desc + " -- expert parallel" + (", one batch split over the GPUs" if strong else ""),
                   "S_total": S_total, "S_per_gpu": S, "TD": TD, "HD": HD, "E": E,
                   "top_k": k, "gating": mode, "experts_per_gpu": El, "placement": args.placement,
                   "parallelism": f"ep{world} ({transport})",
                   "ep_transport": ("p2p" if p2p else "nccl") + (f" -- {transport_note}" if transport_note else ""),
                   "l2": "no flush: per-step local expert weights %.2f GB >> 126 MB L2" % (wbytes / 1e9)},
        "roofline": {"kernel": "whole EP step: local expert weights streamed once per step", "bound": "hbm",
                     "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s", "frac": achieved / hbm_gbs,
                     "peak_kind": peak_kind, "traffic": None},
        "a2a": {"rows_received_rank0": recv_rows, "rows_sent_offrank_rank0": sent_off,
                "payload_bytes_offrank_per_direction": sent_off * TD * 2,
                "exchange_bytes_offrank_per_step": xbytes,
                "exchange_gbs_over_whole_step": xbytes / (ms * 1e-3) / 1e9,
                "nvlink_peak_gbs_per_direction": 900.0,
                "nvlink_peer_copy_gbs_profiling_guide": 770.0,  # B200_PROFILING.md measured figure, not this run
                **({"dispatch_ms": ep_stage["dispatch"], "combine_ms": ep_stage["combine"],
                    "dispatch_gbs_offrank": sent_off * TD * 2 / (ep_stage["dispatch"] * 1e-3) / 1e9,
                    "combine_gbs_offrank": sent_off * TD * 2 / (ep_stage["combine"] * 1e-3) / 1e9,
                    "note": ("dispatch / combine kernel times include the wait for the slowest peer" if p2p else
                             "nccl: dispatch = gather + payload send/recv, combine = weighted combine; "
                             "the return send/recv is in stage 'done'")}
                   if ep_stage else {})},
        "stage_ms": ep_stage,
        "balance": balance,
        "gpu_launches": n_launch * K,
        "e2e": {"value": S_total / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": S_total * TD * 2, "d2h_bytes_per_step": S_total * TD * 2,
                "bytes_note": "whole job: every rank uploads its tokens and reads back its outputs",
                "api": ("PeerExpertParallelMoE.forward (moe_ep_forward_graph)" if p2p else
                        "PeerExpertParallelMoE(transport='nccl').forward (moe_ep_forward, NCCL)")
                       + " (pinned host in/out)"},
        "cpu_baseline": None,
        "clocks": sampler.summary() if sampler else None,
        "gpu": torch.cuda.get_device_name(local),
    }
    emit(line, args)
    layer.close()


def run_cache(args):
    """configs[4]: expert buffering.  All E experts in pinned host memory, a
    LIFO cache of --cache-slots on the GPU; each step is one decoder batch with
    routing from the reference's skewed generator (zipf 1.2, persistence 0.9,
    active fraction 0.75 -- proj/README.md:59-61); the fully resident layer on
    the same batches is timed beside it."""
    import numpy as np
    import torch

    from paper_2303_06182_b200.layer import ExpertCache, LayerShape, MoeLayer, make_tokens, make_weights
    from paper_2303_06182_b200.traces import skewed_routing

    S, TD, HD, E, k, mode, C, desc = WORKLOADS[args.workload]
    S = args.tokens or S
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=2303061820)
    Wg = w[0]
    x = make_tokens(S, TD, seed=2303061821)
    K, W = args.steps, args.warmup
    ex, wt = skewed_routing(E, k, W + K, S, 1.2, 0.9, 0.75, seed=7)
    idx = torch.from_numpy(ex).cuda()
    gw = torch.from_numpy(wt.astype(np.float32)).cuda()
    slots = args.cache_slots or E // 4
    W1h, W2h = w[1].cpu().pin_memory(), w[2].cpu().pin_memory()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
    out = torch.empty_like(x)
    # measured host->device peak of this box: pinned 1 GiB copy, best of 5
    hbuf = torch.empty(1 << 29, dtype=torch.bfloat16).pin_memory()
    dbuf = torch.empty_like(hbuf, device="cuda")
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            dbuf.copy_(hbuf, non_blocking=True)
            e1.record(stream)
        stream.synchronize()
        best = max(best, hbuf.numel() * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    h2d_peak = best
    del hbuf, dbuf
    def timed(fn, after_warmup=None):
        with torch.cuda.stream(stream):
            for b in range(W):
                fn(b)
        stream.synchronize()
        if after_warmup:
            after_warmup()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        with torch.cuda.stream(stream):
            for i in range(K):
                evs[i].record(stream)
                fn(W + i)
            evs[K].record(stream)
        stream.synchronize()
        return [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]

    # fully resident layer on the same batches (all E experts in HBM), then
    # freed: the cached layer holds only the slot pool
    full = MoeLayer(shape, S, weights=w)
    t_full = timed(lambda b: full.forward_routed(x, idx[b], gw[b], out, stream))
    full.close()
    del full, w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    used0 = torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]
    layer = MoeLayer(shape, S, weights=(Wg, None, None), pool_only=True)
    cache = ExpertCache(layer, slots, "lifo", W1h, W2h)
    torch.cuda.synchronize()
    used1 = torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]
    stats0 = {}
    t_cache = timed(lambda b: cache.forward_routed(x, idx[b], gw[b], out, stream),
                    after_warmup=lambda: stats0.update(cache.stats()))  # timed steps only
    s0 = stats0
    s1 = cache.stats()
    acc = s1["accesses"] - s0["accesses"]
    miss = s1["misses"] - s0["misses"]
    copied = s1["bytes_copied"] - s0["bytes_copied"]
    ms = float(np.mean(t_cache))
    expert_bytes = 2 * TD * HD * 2
    line = {
        "metric": "MoE-layer tokens/s (dynamic gating, expert buffering)", "value": S / (ms * 1e-3),
        "unit": "tokens/s", "n_gpus": 1, "steps": K, "warmup": W, "ms_per_step": ms,
        "p50_ms": float(np.median(t_cache)), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic tokens, skewed synthetic routing (reference generator), random-init experts",
        "config": {"workload": desc, "S": S, "TD": TD, "HD": HD, "E": E, "top_k": k, "cache_slots": slots,
                   "policy": "LIFO", "expert_mb": expert_bytes / 2**20},
        "cache": {"accesses": acc, "misses": miss, "miss_rate": miss / max(acc, 1),
                  "active_per_step": acc / K, "h2d_gb_per_step": copied / K / 1e9,
                  "h2d_gbs_achieved": copied / (sum(t_cache) * 1e-3) / 1e9,
                  "h2d_peak_gbs_measured": h2d_peak,
                  "pcie_frac": copied / (sum(t_cache) * 1e-3) / 1e9 / h2d_peak,
                  "copy_bound_ms_per_step": copied / K / (h2d_peak * 1e9) * 1e3,
                  "gpu_expert_memory_gb": slots * expert_bytes / 1e9,
                  "device_memory_of_cached_layer_gb": (used1 - used0) / 1e9,
                  "resident_expert_memory_gb": E * expert_bytes / 1e9},
        "fully_resident": {"ms_per_step": float(np.mean(t_full)), "value": S / (np.mean(t_full) * 1e-3)},
        "gpu": torch.cuda.get_device_name(0),
    }
    emit(line, args)
    cache.close()


def run_b200(args):
    import numpy as np
    import torch

    from paper_2303_06182_b200 import _capi
    from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    if args.workload == "mt-cache":
        run_cache(args)
        return
    if world > 1 and not args.replicas:
        run_ep(args, world, rank, local)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    S, TD, HD, E, k, mode, C, desc = WORKLOADS[args.workload]
    hbm_gbs, tflops, peak_kind = measured_peaks()
    shape = LayerShape(TD, HD, E, k)
    seed = 2303061820 + rank
    weights = make_weights(shape, seed=2303061820)
    # expert weights held ONCE: the dynamic-gating layer streams them tile-packed
    # in place (no second copy); static gating streams them row-major
    in_place = mode == "dynamic" and not args.split_ffn
    torch.cuda.synchronize()
    free0, total_mem = torch.cuda.mem_get_info()
    layer = MoeLayer(shape, S, mode=mode, capacity_factor=C if mode == "static" else 1.0, weights=weights,
                     tile_n=args.tile_n, fuse_combine=args.fuse_combine,
                     split_ffn=args.split_ffn, pack_in_place=in_place)
    del weights
    torch.cuda.synchronize()
    expert_bytes = E * 2 * TD * HD * 2
    mem = {"expert_weight_bytes": expert_bytes,
           "expert_weight_copies_in_hbm": 1 if (in_place or mode == "static") else 2,
           "layer_extra_device_bytes": free0 - torch.cuda.mem_get_info()[0],
           "device_used_gb": (total_mem - torch.cuda.mem_get_info()[0]) / 1e9}
    x = make_tokens(S, TD, seed=seed)
    out = torch.empty_like(x)
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
    lib = layer.ctx.lib
    K, W = args.steps, args.warmup
    _capi.check(lib.moe_layer_enable_timing(layer.h, 0))

    with torch.cuda.stream(stream):
        for _ in range(W):
            layer.forward(x, out, stream=stream)
    stream.synchronize()
    layer.check_errors(stream)
    v = layer.view()
    counts = v["counts"].cpu().numpy()
    active = int((counts > 0).sum()) if mode == "dynamic" else E
    rows = int(v["rows"])
    import ctypes

    # ---- per-stage breakdown (CUDA events between the kernels of each step),
    #      a separate pass: event records between kernels would break the
    #      programmatic-dependent-launch overlap of the timed steps
    Ks = min(K, 20)
    _capi.check(lib.moe_layer_enable_timing(layer.h, Ks))
    with torch.cuda.stream(stream):
        for _ in range(Ks):
            layer.forward(x, out, stream=stream)
    stream.synchronize()
    stage = np.zeros((Ks, len(STAGES)), np.float64)
    buf = (ctypes.c_float * len(STAGES))()
    for i in range(Ks):
        _capi.check(lib.moe_layer_stage_times(layer.h, i, ctypes.cast(buf, ctypes.c_void_p)))
        stage[i] = list(buf)
    _capi.check(lib.moe_layer_enable_timing(layer.h, 0))

    # ---- timed region: K steps (one CUDA-graph replay of the whole layer per
    #      step unless --no-graph), events per step for the p50
    use_graph = not args.no_graph
    with torch.cuda.stream(stream):
        for _ in range(2):
            layer.forward(x, out, graph=use_graph, stream=stream)
    stream.synchronize()

    def timed_region():
        sampler = ClockSampler(local) if not args.no_clocks else None
        if sampler:
            sampler.start()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        barrier(world)
        torch.cuda.synchronize()
        if sampler:
            sampler.mark_start()
        with torch.cuda.stream(stream):
            for i in range(K):
                evs[i].record(stream)
                layer.forward(x, out, graph=use_graph, stream=stream)
            evs[K].record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        if sampler:
            sampler.mark_stop()
        barrier(world)
        layer.check_errors(stream)
        if sampler:
            sampler.stop()
        return (evs[0].elapsed_time(evs[K]), np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(K)]),
                sampler.summary() if sampler else None)

    elapsed_ms, step_ms, clocks = timed_region()
    # a timed region that saw hardware / thermal slowdown is measured again once
    # (sw_power_cap is normal for a 1 kW part and kept)
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    throttled = bool(clocks and bad & set(clocks.get("reasons", [])))
    remeasured = None
    if max_over_ranks(1.0 if throttled else 0.0, world) > 0:
        remeasured = {"first_attempt_reasons": clocks.get("reasons") if clocks else None,
                      "first_attempt_ms_per_step": elapsed_ms / K}
        elapsed_ms, step_ms, clocks = timed_region()
    elapsed_max = max_over_ranks(elapsed_ms, world)
    p50 = float(np.median(step_ms))
    p50_max = max_over_ranks(p50, world)
    p90_max = max_over_ranks(float(np.percentile(step_ms, 90)), world)
    if remeasured and clocks is not None:
        clocks = dict(clocks, remeasured=remeasured)

    # ---- e2e through the public C-ABI host path (pinned host in/out, copies in the timed region)
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    Ke = max(3, min(K, args.e2e_steps))
    for _ in range(2):
        layer.forward_host(xh, oh, stream=stream)
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call_ms = []
    for _ in range(Ke):
        tc = time.perf_counter()
        layer.forward_host(xh, oh, stream=stream)  # returns after the read-back
        call_ms.append((time.perf_counter() - tc) * 1e3)
    e1.record(stream)
    e1.synchronize()
    e2e_sync_ms = max_over_ranks(e0.elapsed_time(e1) / Ke, world)
    call_p50_ms = max_over_ranks(float(np.median(call_ms)), world)
    # serving queue: Ke batches, each uploaded from and read back to its own
    # pinned host buffers (ring of 3 distinct token sets), copies overlapped
    # with the neighbouring batches' compute (moe_layer_forward_host_batches)
    ring_x = [xh] + [make_tokens(S, TD, seed=seed + 1000 + r).cpu().pin_memory() for r in range(2)]
    ring_o = [torch.empty_like(xh).pin_memory() for _ in range(3)]
    xs = [ring_x[i % 3] for i in range(Ke)]
    os_ = [ring_o[i % 3] for i in range(Ke)]
    layer.forward_host_batches(xs[:3], os_[:3], stream)
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(stream)
    layer.forward_host_batches(xs, os_, stream)  # synchronous: returns after the last read-back
    e1.record(stream)
    e1.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3 / Ke
    e2e_dev_ms = e0.elapsed_time(e1) / Ke
    e2e_ms = max_over_ranks(max(e2e_dev_ms, wall_ms), world)
    if not torch.equal(ring_o[0], oh):
        raise RuntimeError("pipelined host path differs from moe_layer_forward_host")

    if rank != 0:
        return
    ms_per_step = elapsed_max / K
    value = world * S / (ms_per_step * 1e-3)
    mean_stage = stage.mean(0)
    one_launch = ((mode == "dynamic" or os.environ.get("MOE_FUSED_STATIC", "1") != "0")
                  and int(v["tile_n"]) in (128, 256) and not args.split_ffn
                  and (int(v["tile_n"]) == 128 or os.environ.get("MOE_FUSED_256", "1") != "0"))
    launches_per_step = (3 + (1 if one_launch else 2)
                         + (0 if args.fuse_combine else 1))
    ffn_b = ffn_bytes(rows, active, TD, HD, one_launch)
    ffn_ms = mean_stage[3] + mean_stage[4]
    # the FFN's binding roofline: weight/activation bytes at HBM bandwidth, or
    # its MMA flops (4 * rows * TD * HD, static placeholders included) at the
    # tensor peak -- whichever takes longer
    ffn_f = 4.0 * rows * TD * HD
    tensor_bound = ffn_f / (tflops * 1e12) > ffn_b / (hbm_gbs * 1e9)
    if tensor_bound:
        # a multi-ms tensor-bound launch runs under the power cap: sustained peak
        peak_t = sustained_tflops(tflops) if ffn_ms > 1.0 else tflops
        achieved, peak, unit = ffn_f / (ffn_ms * 1e-3) / 1e12, peak_t, "TFLOP/s"
    else:
        achieved, peak, unit = ffn_b / (ffn_ms * 1e-3) / 1e9, hbm_gbs, "GB/s"
    traffic = load_traffic(args.workload) if one_launch else None
    t_roof, F, B = layer_roofline(S, TD, HD, E, k, active, hbm_gbs, tflops)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from oracle.cpu_layer import cpu_layer_bench

        from oracle.cpu_layer import cpu_layer_1thread, routing_1thread

        r = cpu_layer_bench(S, TD, HD, E, k, min_seconds=cpu_seconds())
        cpu = {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": r["cores"], "kind": "port",
               "sample": r["sample"], "breakdown_s": r["breakdown_s"], "cpu_model": r["cpu_model"],
               "host_cpus": r["host_cpus"]}
        if os.environ.get("MOE_BENCH_CPU_DETAIL", "1") != "0":
            # the 1-thread layer and the reference's routing
            # alone (Batch prebuilt, no marshalling) beside the GPU route stage
            cpu["one_thread"] = cpu_layer_1thread(S, TD, HD, E, k)
            cpu["routing_1thread_s"] = routing_1thread(S, TD, E, k, C if mode == "static" else 0.0)
            cpu["routing_1thread_s"]["gpu_route_stage_s"] = float(mean_stage[1]) * 1e-3
    line = {
        "metric": "MoE-layer tokens/s (dynamic gating)" if mode == "dynamic" else "MoE-layer tokens/s (static gating)",
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "p50_ms": p50_max, "p90_ms": p90_max, "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-hash uniform tokens; random-init experts, std 1/sqrt(fan-in))",
        "config": {"workload": desc, "S_per_gpu": S, "TD": TD, "HD": HD, "E": E, "top_k": k, "gating": mode,
                   "capacity_factor": C if mode == "static" else None, "rows": rows, "active_experts": active,
                   "tile_n": int(v["tile_n"]),
                   "parallelism": f"replicas x{world} (all experts on every GPU)" if world > 1 else "single GPU",
                   "l2": "no flush: per-step working set (expert weights, %.1f GB) >> 126 MB L2" % (
                       2 * active * TD * HD * 2 / 1e9)},
        "roofline": {"kernel": {0: "grouped_gemm_kernel (FFN GEMM1 + GEMM2, two launches)",
                                1: "fused_ffn_kernel (GEMM1+GEMM2, one launch, H in L2)",
                                2: "fused_ffn_pair_kernel (GEMM1+GEMM2, one launch, H in L2, CTA pairs: "
                                   "tcgen05.mma.cta_group::2, M=256)"}.get(int(v.get("ffn_kernel", 1)),
                                                                          "fused_ffn_kernel"),
                     "bound": "tensor" if tensor_bound else "hbm",
                     "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                     "peak_kind": peak_kind + (" (sustained)" if tensor_bound and ffn_ms > 1.0 else ""),
                     "algorithmic_bytes_per_step": ffn_b, "algorithmic_flops_per_step": ffn_f,
                     "traffic": traffic,
                     # the peak is MEASURED_PEAKS' copy bandwidth (read + write); a read-only
                     # weight stream can exceed it: its measured ceiling on B200 is
                     # READ_CEILING_GBS (profiles/r01_s2_hbm_read_ceiling.txt)
                     **({"read_ceiling_gbs": READ_CEILING_GBS,
                         "frac_of_read_ceiling": achieved / READ_CEILING_GBS} if not tensor_bound else {})},
        "layer_roofline": {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms_per_step, "flops": F,
                           "bytes": B, "peaks": {"hbm_gbs": hbm_gbs, "bf16_tflops": tflops}},
        "stage_ms": {n: float(m) for n, m in zip(STAGES, mean_stage)},
        "memory": mem,
        "timed_path": "CUDA graph replay of moe_layer_forward (PDL edges)" if use_graph else "eager launches",
        "gpu_launches": launches_per_step * K,
        "e2e": {"value": world * S / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": S * TD * 2, "d2h_bytes_per_step": S * TD * 2,
                "api": ("moe_layer_forward_host_batches (C ABI): %d batches from pinned host buffers, "
                        "upload/compute/read-back pipelined over 3 streams; time = max(device events, "
                        "host wall clock)" % Ke),
                "device_ms_per_step": e2e_dev_ms, "wall_ms_per_step": wall_ms,
                "per_call_sync": {"value": world * S / (e2e_sync_ms * 1e-3), "ms_per_step": e2e_sync_ms,
                                  "p50_ms_wall": call_p50_ms,
                                  "api": "moe_layer_forward_host (one synchronous call per batch)"}},
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu": torch.cuda.get_device_name(local),
    }
    emit(line, args)
    layer.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference", "ours"])
    ap.add_argument("--workload", default="lm", choices=sorted(WORKLOADS))
    ap.add_argument("--tile-n", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=60)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--json-out", default="")
    ap.add_argument("--replicas", action="store_true", help="N>1: full replicas instead of EP")
    ap.add_argument("--placement", default="greedy", choices=["greedy", "contiguous"])
    ap.add_argument("--ep-transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 exchange: NVLink peer memory (fused kernels) or NCCL all-to-all")
    ap.add_argument("--cache-slots", type=int, default=0, help="mt-cache: GPU slots (default E/4)")
    ap.add_argument("--tokens", type=int, default=0, help="override tokens per step (mt-cache)")
    ap.add_argument("--fuse-combine", action="store_true", help="combine in the GEMM2 epilogue (A/B)")
    ap.add_argument("--split-ffn", action="store_true", help="GEMM1/GEMM2 as two launches (A/B)")
    ap.add_argument("--no-graph", action="store_true", help="timed steps as eager launches")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = S tokens per GPU; strong = S tokens in total, split over the GPUs "
                         "(configs[3]: the LM batch of 16384 tokens across 2/4/8 GPUs)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch / rendezvous check only: every rank prints its world and rank, no GPU work")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl != "reference" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` outside torchrun: relaunch as N ranks (one process per GPU)
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        # every rank prints here
        _write_line(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": args.gpus, "world": world,
                                "rank": int(os.environ.get("RANK", "0")), "scaling": args.scaling}))
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
