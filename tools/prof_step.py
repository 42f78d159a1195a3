"""Minimal step runner for ncu captures (eager launches, no timing).

  python tools/prof_step.py [--workload lm|mt|cfg1] [--steps N] [--ep]

--ep runs the expert-parallel layer with the peer-memory exchange at world
size 1 (moe_ep_*: publish / dispatch / recv / FFN / done / combine kernels).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS  # noqa: E402
from paper_2303_06182_b200.layer import Context, LayerShape, MoeLayer, make_tokens, make_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="lm")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--ep", action="store_true")
ap.add_argument("--tile-n", type=int, default=0)
a = ap.parse_args()
S, TD, HD, E, k, mode, C, _ = WORKLOADS[a.workload]
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape)
x = make_tokens(S, TD)
out = torch.empty_like(x)
if a.ep:
    from paper_2303_06182_b200.ep import PeerExpertParallelMoE, Placement

    layer = PeerExpertParallelMoE(Context.get(0), Placement.contiguous(E, 1), shape, w[0], w[1], w[2], S, 0)
    for _ in range(a.steps):
        layer.forward(x, out=out)
    layer.check_errors()
else:
    layer = MoeLayer(shape, S, mode=mode, capacity_factor=C or 1.0, weights=w, tile_n=a.tile_n)
    for _ in range(a.steps):
        layer.forward(x, out)
    layer.check_errors()
torch.cuda.synchronize()
print("ok")
