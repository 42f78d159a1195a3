import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights
SEED = 2303061820
S, TD, HD, E, k = 16384, 1024, 4096, 512, 2
shape = LayerShape(TD, HD, E, k)
w = make_weights(shape, seed=SEED)
x = make_tokens(S, TD, seed=SEED)
ref_layer = MoeLayer(shape, S, weights=w, split_ffn=True, keep_logits=True)
ref = ref_layer(x); torch.cuda.synchronize()
ref2 = ref_layer(x); torch.cuda.synchronize()
print("split deterministic:", torch.equal(ref, ref2))
rv = ref_layer.view()
idx_ref = rv["idx"][:S*k].clone()
layer = MoeLayer(shape, S, weights=w, keep_logits=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
def report(name, out):
    bad = (out != ref).any(1).nonzero().flatten()
    v = layer.view()
    idx_ok = torch.equal(v["idx"][:S*k], idx_ref)
    print(f"{name}: bad rows {bad.numel()} first {bad[:8].tolist()} idx_equal={idx_ok}", flush=True)
for trial in range(6):
    with torch.cuda.stream(s):
        out = layer(x, stream=s)
    s.synchronize()
    report(f"eager{trial}", out)
with torch.cuda.stream(s):
    out_g = torch.empty_like(x)
    for trial in range(4):
        layer.forward(x, out_g, graph=True, stream=s)
        s.synchronize()
        report(f"graph{trial}", out_g)
