"""Does running consecutive batches on two streams (independent layer
buffers) fill the FFN tail / overlap the front with the previous FFN?
Experiment only: two full MoeLayer instances."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights  # noqa: E402

S, TD, HD, E, k = 16384, 1024, 4096, 512, 2
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape)
x = make_tokens(S, TD)
nl = int(sys.argv[1]) if len(sys.argv) > 1 else 2
layers = [MoeLayer(shape, S, weights=w) for _ in range(nl)]
outs = [torch.empty_like(x) for _ in range(nl)]
streams = [torch.cuda.Stream() for _ in range(nl)]
main = torch.cuda.current_stream()
K = 60


def run(n_streams):
    for s in streams:
        s.wait_stream(main)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(6):
        j = i % n_streams
        layers[j].forward(x, outs[j], graph=True, stream=streams[j])
    for s in streams:
        main.wait_stream(s)
    torch.cuda.synchronize()
    a.record(main)
    for s in streams:
        s.wait_stream(main)
    for i in range(K):
        j = i % n_streams
        layers[j].forward(x, outs[j], graph=True, stream=streams[j])
    for s in streams:
        main.wait_stream(s)
    b.record(main)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


for rep in range(2):
    for n in range(1, nl + 1):
        print(f"streams={n}: {run(n):.4f} ms/batch", flush=True)
ref = outs[0].clone()
run(nl)
torch.cuda.synchronize()
print("outputs equal:", all(bool((o == ref).all()) for o in outs))
