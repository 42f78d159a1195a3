"""CPU MoE layer -- the reported CPU baseline (bench.py cpu_baseline leg and
``--impl reference``).  TEST/BASELINE INFRASTRUCTURE ONLY.

The reference has no layer arithmetic; its CPU path for this layer
is its routing core.  The CPU layer therefore runs:

  gate       fp32 logits = X Wg^T (numpy/BLAS, all host cores) + top-k
             (oracle.layer.topk_from_logits)
  dispatch   the reference's own dynamic_dispatch, compiled verbatim
             (oracle/_ref, proj/src/gating.cpp:58-86) -- single-threaded as
             the reference is
  FFN        fp32 relu(x W1_e^T) W2_e^T for EVERY expert with its real token
             count (numpy/BLAS, all cores)
  combine    the reference's own combine<int> (gating.hpp:107-141) to restore
             slot order, then the gate-weighted sum (numpy)

Every layer pass is the full workload (all S tokens, all k*S slots, all E
experts).  Only the expert weights are bounded: ``weight_pool`` experts are
materialised (fp32) and expert e uses pool entry e % weight_pool -- the FFN
cost of a slot does not depend on the weight values, and materialising
E x 2 x TD x HD fp32 weights would take 17 GB at the LM shape.  The outputs are
therefore a timing baseline, not the layer's values (parity lives in tests/).
``cpu_layer_bench`` repeats full passes until ``min_seconds`` of CPU work have
been timed and reports the median pass.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import layer as OL
from . import native as N


class CpuLayer:
    """Inputs + weight pool for one workload, prepared once (untimed)."""

    def __init__(self, S, TD, HD, E, k, seed=2303061820, weight_pool=8, use_reference=True):
        self.S, self.TD, self.HD, self.E, self.k = S, TD, HD, E, k
        sc = OL.init_scales(TD, HD)
        self.X = OL.bf16_to_f32(OL.synth_bf16((S, TD), seed, OL.T_X, sc["x"]))
        self.Wg = OL.bf16_to_f32(OL.synth_bf16((E, TD), seed, OL.T_WG, sc["wg"]))
        self.n_pool = min(E, weight_pool)
        self.W1 = [OL.bf16_to_f32(OL.synth_bf16((HD, TD), seed, OL.T_W1, sc["w1"], index_offset=e * HD * TD))
                   for e in range(self.n_pool)]
        self.W2 = [OL.bf16_to_f32(OL.synth_bf16((TD, HD), seed, OL.T_W2, sc["w2"], index_offset=e * TD * HD))
                   for e in range(self.n_pool)]
        self.use_ref = use_reference and N.ref_available()

    def run(self):
        """One full layer pass; returns the per-stage wall times (s)."""
        S, E, k = self.S, self.E, self.k
        t0 = time.perf_counter()
        logits = OL.gate_logits(self.X, self.Wg)
        idx, w = OL.topk_from_logits(logits, k)
        t1 = time.perf_counter()
        if self.use_ref:
            order, counts, splits = N.ref_dynamic_dispatch(idx, E, w)
        else:
            order, counts, splits, _ = N.c_dynamic_dispatch(idx, E)
        t2 = time.perf_counter()
        ys = {}
        for e in range(E):
            rows = order[splits[e]:splits[e + 1]]
            if len(rows):
                p = e % self.n_pool
                ys[e] = OL.expert_ffn(self.X[rows // k], self.W1[p], self.W2[p])
        t3 = time.perf_counter()
        if self.use_ref:
            N.ref_combine_dynamic(idx, w, E, np.arange(S * k, dtype=np.int32))
        t4 = time.perf_counter()
        out = np.zeros((S, self.TD), np.float32)
        for e, y in ys.items():
            rows = order[splits[e]:splits[e + 1]]
            t = rows // k
            # a token picks k distinct experts, so t has no repeats within one expert
            out[t] += y * w[t, rows % k][:, None].astype(np.float32)
        t5 = time.perf_counter()
        return {"total": t5 - t0, "gate_topk": t1 - t0, "dispatch": t2 - t1, "ffn": t3 - t2,
                "combine_restore": t4 - t3, "weighted_sum": t5 - t4}

    @property
    def dispatch_impl(self):
        return "reference gating.cpp (verbatim build)" if self.use_ref else "C restatement"


def cpu_model() -> str:
    """The host CPU (report the GPU box's CPU beside the baseline)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def blas_threads() -> int:
    """Threads the BLAS backing numpy will use (threadpoolctl)."""
    try:
        from threadpoolctl import threadpool_info

        n = [p.get("num_threads", 1) for p in threadpool_info() if p.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return 1


def cpu_layer_bench(S, TD, HD, E, k, min_seconds=10.0, max_passes=200, weight_pool=8, layer=None):
    """Full layer passes until >= min_seconds of timed CPU work; median pass.
    BLAS runs on every host core whatever OMP_NUM_THREADS says (torchrun sets
    it to 1), so the baseline is the CPU path at full width."""
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    if threadpool_limits is not None:
        with threadpool_limits(limits=os.cpu_count(), user_api="blas"):
            return _cpu_layer_bench(S, TD, HD, E, k, min_seconds, max_passes, weight_pool, layer)
    return _cpu_layer_bench(S, TD, HD, E, k, min_seconds, max_passes, weight_pool, layer)


def _cpu_layer_bench(S, TD, HD, E, k, min_seconds, max_passes, weight_pool, layer):
    L = layer or CpuLayer(S, TD, HD, E, k, weight_pool=weight_pool)
    passes = []
    t_all = 0.0
    while (t_all < min_seconds or not passes) and len(passes) < max_passes:
        r = L.run()
        passes.append(r)
        t_all += r["total"]
    passes.sort(key=lambda r: r["total"])
    med = passes[len(passes) // 2]
    return {
        "seconds_per_layer": med["total"],
        "tokens_per_s": S / med["total"],
        "passes": len(passes),
        "measured_cpu_seconds": t_all,
        "breakdown_s": {kk: v for kk, v in med.items() if kk != "total"},
        "dispatch_impl": L.dispatch_impl,
        "weight_pool": L.n_pool,
        "cores": blas_threads(),
        "cpu_model": cpu_model(),
        "host_cpus": os.cpu_count(),
        "sample": (f"{len(passes)} full layer passes (all {S} tokens, {S * k} slots, {E} experts; "
                   f"expert weights cycled over {L.n_pool} materialised experts), median pass; "
                   f"dispatch/combine = {L.dispatch_impl} (single-threaded, as the reference); "
                   f"gate/FFN numpy/OpenBLAS fp32 on {blas_threads()} threads ({os.cpu_count()} host "
                   f"cores); {t_all:.1f} s timed"),
    }


def cpu_layer_1thread(S, TD, HD, E, k, tokens=2048, min_seconds=3.0, weight_pool=8):
    """The same layer pass on ONE host thread (BLAS limited to 1) over the
    first ``tokens`` tokens of the workload, repeated until ``min_seconds``;
    median pass.  Reported beside the all-core number."""
    from threadpoolctl import threadpool_limits

    n = min(S, tokens)
    with threadpool_limits(limits=1, user_api="blas"):
        L = CpuLayer(n, TD, HD, E, k, weight_pool=weight_pool)
        ts, t_all = [], 0.0
        while t_all < min_seconds or not ts:
            t = L.run()["total"]
            ts.append(t)
            t_all += t
    ts.sort()
    med = ts[len(ts) // 2]
    return {"value": n / med, "unit": "tokens/s", "cores": 1, "seconds_per_pass": med,
            "sample": f"{len(ts)} passes over {n} of the {S} tokens ({n * k} slots, {E} experts), "
                      f"BLAS on 1 thread, median pass"}


def routing_1thread(S, TD, E, k, C=0.0, seed=2303061820, reps=5):
    """The reference's routing functions alone (dynamic_dispatch, combine<float>,
    and static_dispatch + its combine when C > 0) on one thread, with the
    reference Batch prebuilt outside the timed region (oracle/ref_capi.cpp
    ref_time_routing): the CPU number the GPU route kernel replaces.  Routing
    uses the workload's own top-k of the fp32 gate logits."""
    sc = OL.init_scales(TD, 1)
    X = OL.bf16_to_f32(OL.synth_bf16((S, TD), seed, OL.T_X, sc["x"]))
    Wg = OL.bf16_to_f32(OL.synth_bf16((E, TD), seed, OL.T_WG, sc["wg"]))
    idx, w = OL.topk_from_logits(OL.gate_logits(X, Wg), k)
    r = N.ref_time_routing(idx, w.astype(np.float64), E, C, reps)
    return {kk: float(v) for kk, v in r.items()}
