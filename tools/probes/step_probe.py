"""Where does a step go?  K forwards timed with two events only, eager vs graph."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights  # noqa: E402

S, TD, HD, E, k = 16384, 1024, 4096, 512, 2
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape)
x = make_tokens(S, TD)
layer = MoeLayer(shape, S, weights=w)
out = torch.empty_like(x)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
K = 100
for graph in (False, True, False, True):
    with torch.cuda.stream(s):
        for _ in range(5):
            layer.forward(x, out, graph=graph, stream=s)
    s.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(K):
            layer.forward(x, out, graph=graph, stream=s)
        b.record(s)
    s.synchronize()
    print("graph" if graph else "eager", round(a.elapsed_time(b) / K, 4), "ms/step")
