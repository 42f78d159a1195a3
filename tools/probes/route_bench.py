"""Micro-benchmark of the route kernel (moe_route_dynamic) with CUDA events."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2303_06182_b200.layer import Context, _stream_ptr  # noqa: E402

ctx = Context.get(0)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for S, E, k in [(2048, 8, 1), (16384, 512, 2), (6144, 128, 2), (131072, 512, 2)]:
    idx = torch.randint(0, E, (S * k,), dtype=torch.int32, device="cuda")
    counts = torch.empty(E, dtype=torch.int32, device="cuda")
    splits = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    order = torch.empty(S * k, dtype=torch.int32, device="cuda")
    pos = torch.empty(S * k, dtype=torch.int32, device="cuda")
    for _ in range(5):
        ctx.lib.moe_route_dynamic(ctx.h, P(idx), S, k, E, P(counts), P(splits), P(order), P(pos), _stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 50
    for _ in range(n):
        ctx.lib.moe_route_dynamic(ctx.h, P(idx), S, k, E, P(counts), P(splits), P(order), P(pos), _stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    print(f"route S={S} E={E} k={k}: {e0.elapsed_time(e1) / n * 1000:.1f} us/call")
