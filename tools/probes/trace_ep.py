"""GPU timeline of expert-parallel steps at world 1 (graph replay), CUPTI."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2303_06182_b200.ep import PeerExpertParallelMoE, Placement  # noqa: E402
from paper_2303_06182_b200.layer import Context, LayerShape, make_tokens, make_weights  # noqa: E402

S, TD, HD, E, k = 16384, 1024, 4096, 512, 2
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape)
x = make_tokens(S, TD)
out = torch.empty_like(x)
ep = PeerExpertParallelMoE(Context.get(0), Placement.contiguous(E, 1), shape, w[0], w[1], w[2], S, 0)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(5):
        ep.forward(x, stream=s, out=out, graph=True)
s.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(s):
        for _ in range(3):
            ep.forward(x, stream=s, out=out, graph=True)
    s.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = None
for e in ev:
    st, en = e.time_range.start - t0, e.time_range.end - t0
    print(f"{st:10.1f} {en - st:9.1f} us {'' if prev is None else f'gap {st - prev:8.1f}'}  {e.name[:60]}")
    prev = en
