import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights
for (S, TD, HD, E, k) in [(16384, 1024, 4096, 512, 2), (2048, 1024, 4096, 8, 1), (6144, 2048, 8192, 128, 2), (3000, 256, 512, 40, 3)]:
    shape = LayerShape(TD, HD, E, k)
    L = MoeLayer(shape, S, weights=make_weights(shape))
    x = make_tokens(S, TD)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        o1 = L(x, stream=s).clone()
        o2 = L(x, graph=True, stream=s).clone()
    s.synchronize()
    np.save(f"{sys.argv[1]}_{S}_{E}.npy", o2.view(torch.int16).cpu().numpy())
    print(S, E, "eager==graph", torch.equal(o1, o2))
    L.close()
