"""GPU timeline of a few layer steps (torch.profiler / CUPTI activity trace):
kernel start/end per step and the gaps between them."""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "lm"
S, TD, HD, E, k = {"lm": (16384, 1024, 4096, 512, 2), "cfg1": (2048, 1024, 4096, 8, 1)}[wl]
graph = "graph" in sys.argv
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape)
x = make_tokens(S, TD)
layer = MoeLayer(shape, S, weights=w)
out = torch.empty_like(x)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
with torch.cuda.stream(s):
    for _ in range(5):
        layer.forward(x, out, graph=graph, stream=s)
s.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(s):
        for _ in range(4):
            layer.forward(x, out, graph=graph, stream=s)
    s.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = None
for e in ev:
    st, en = e.time_range.start - t0, e.time_range.end - t0
    gap = "" if prev_end is None else f"gap {st - prev_end:8.1f}"
    print(f"{st:10.1f} {en - st:9.1f} us {gap}  {e.name[:70]}")
    prev_end = en
