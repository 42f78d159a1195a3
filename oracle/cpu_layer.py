"""CPU MoE layer -- the reported CPU baseline (bench.py cpu_baseline leg and
``--impl reference``).  TEST/BASELINE INFRASTRUCTURE ONLY.

The reference has no layer arithmetic; its CPU path for this layer
is its routing core.  The CPU layer therefore runs:

  gate       fp32 logits = X Wg^T (numpy/BLAS, all host cores) + top-k
             (oracle.layer.topk_from_logits)
  dispatch   the reference's own dynamic_dispatch, compiled verbatim
             (oracle/_ref, proj/src/gating.cpp:58-86) -- single-threaded as
             the reference is
  FFN        fp32 relu(x W1_e^T) W2_e^T per expert (numpy/BLAS, all cores)
  combine    the reference's own combine<int> (gating.hpp:107-141) to restore
             slot order, then the gate-weighted sum (numpy)

Bounded sample: the gate, dispatch and combine run on the FULL batch; the
expert FFN runs for the first ``n_sample_experts`` experts with their real
token counts (weights for only those experts are materialised), and its time
is scaled by total_slots / sampled_slots.  The FFN cost per slot does not
depend on which expert serves it, so this estimates the full-batch time
without generating E x 2 x TD x HD fp32 weights (17 GB at the LM shape).
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import layer as OL
from . import native as N


def cpu_layer_sample(S, TD, HD, E, k, seed=2303061820, n_sample_experts=8, use_reference=True):
    sc = OL.init_scales(TD, HD)
    X = OL.bf16_to_f32(OL.synth_bf16((S, TD), seed, OL.T_X, sc["x"]))
    Wg = OL.bf16_to_f32(OL.synth_bf16((E, TD), seed, OL.T_WG, sc["wg"]))
    n_se = min(E, n_sample_experts)
    W1 = [OL.bf16_to_f32(OL.synth_bf16((HD, TD), seed, OL.T_W1, sc["w1"], index_offset=e * HD * TD))
          for e in range(n_se)]
    W2 = [OL.bf16_to_f32(OL.synth_bf16((TD, HD), seed, OL.T_W2, sc["w2"], index_offset=e * TD * HD))
          for e in range(n_se)]

    t0 = time.perf_counter()
    logits = OL.gate_logits(X, Wg)
    idx, w = OL.topk_from_logits(logits, k)
    t1 = time.perf_counter()
    if use_reference and N.ref_available():
        order, counts, splits = N.ref_dynamic_dispatch(idx, E, w)
        dispatch_impl = "reference gating.cpp (verbatim build)"
    else:
        order, counts, splits, _ = N.c_dynamic_dispatch(idx, E)
        dispatch_impl = "C restatement"
    t2 = time.perf_counter()
    ys = {}
    sampled = 0
    for e in range(n_se):
        rows = order[splits[e]:splits[e + 1]]
        if len(rows) == 0:
            continue
        ys[e] = OL.expert_ffn(X[rows // k], W1[e], W2[e])
        sampled += len(rows)
    t3 = time.perf_counter()
    # combine: reference restores slot order, then the weighted sum
    if use_reference and N.ref_available():
        n, oe, ow, op = N.ref_combine_dynamic(idx, w, E, np.arange(S * k, dtype=np.int32))
    else:
        op = None
    t4 = time.perf_counter()
    out = np.zeros((S, TD), np.float32)
    done = 0
    for e, y in ys.items():
        rows = order[splits[e]:splits[e + 1]]
        t = rows // k
        j = rows % k
        # a token picks k distinct experts, so t has no repeats within one expert
        out[t] += y * w[t, j][:, None].astype(np.float32)
        done += len(rows)
    t5 = time.perf_counter()

    total_slots = S * k
    scale = total_slots / max(sampled, 1)
    ffn = (t3 - t2) * scale
    wsum = (t5 - t4) * scale
    total = (t1 - t0) + (t2 - t1) + ffn + (t4 - t3) + wsum
    return {
        "seconds_per_layer": total,
        "tokens_per_s": S / total,
        "breakdown_s": {"gate_topk": t1 - t0, "dispatch": t2 - t1, "ffn_est": ffn,
                        "combine_restore": t4 - t3, "weighted_sum_est": wsum},
        "sampled_slots": int(sampled), "total_slots": int(total_slots),
        "measured_cpu_seconds": (t5 - t0),
        "dispatch_impl": dispatch_impl,
        "cores": os.cpu_count(),
    }
