"""Small-shape runs of every kernel family, for compute-sanitizer
(tools/sanitize.sh runs each case under memcheck, racecheck and synccheck).

  python tools/sanitize_cases.py <case>

Cases (eager launches, one or two forwards each, outputs checked against the
fp32 oracle so a sanitizer-clean run is also a correct one):
  cfg1     E=8 top-1: split-K cluster gate, one-CTA route, 1-SM fused FFN
  lm       E=512 top-2: 32-deep gate (E > 128), grid route, CTA-pair FFN
  mt256    E=128 top-2, tile_n=256: wide gate, 256-token CTA-pair FFN items
  onesm    E=64 top-2 with CTA pairs off: the 1-SM fused FFN at tile_n 128
  split    E=64 top-2, split FFN (grouped_gemm_kernel GEMM1 + GEMM2)
  static   E=16 top-2 static gating CF=1 (capacity clip, drop marks)
  route    route kernel alone: one-CTA form and the grid form, 40k slots
  cache    E=32 top-2 through a 6-slot LIFO expert cache (pool-only layer)
  host     moe_layer_forward_host + forward_host_batches (3 staging streams)
  ep1      expert parallel at world 1 (publish/dispatch/recv/FFN/done/combine)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import layer as OL  # noqa: E402  (checker only)
from paper_2303_06182_b200.layer import (Context, ExpertCache, LayerShape, MoeLayer,  # noqa: E402
                                         make_tokens, make_weights)


def run_layer(S, TD, HD, E, k, mode="dynamic", C=1.0, tile_n=0, split=False, graph=False):
    shape = LayerShape(TD, HD, E, k)
    W = make_weights(shape)
    x = make_tokens(S, TD)
    L = MoeLayer(shape, S, mode=mode, capacity_factor=C, weights=W, tile_n=tile_n, split_ffn=split)
    out = L(x)
    out = L(x, graph=graph, stream=torch.cuda.current_stream())
    L.check_errors()
    torch.cuda.synchronize()
    v = L.view()
    idx = v["idx"].reshape(-1, k)[:S].cpu().numpy()
    w = v["w"].reshape(-1, k)[:S].cpu().numpy()
    toks = np.unique(np.linspace(0, S - 1, 48).astype(int))
    X = x.float().cpu().numpy()
    W1 = W[1].float().cpu().numpy()
    W2 = W[2].float().cpu().numpy()
    if mode == "static":
        ref = _static_ref(X, W1, W2, idx, w, E, k, C, toks)
    else:
        ref = OL.layer_forward(X, W1, W2, idx, w, E, tokens=toks)
    got = out.float().cpu().numpy()[toks]
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-6)
    print(f"S={S} TD={TD} HD={HD} E={E} k={k} {mode} tile_n={L.view().get('tile_n', tile_n)}: "
          f"max|d|/max|ref| = {err:.2e}")
    assert err < 2e-2, err
    L.close()


def _static_ref(X, W1, W2, idx, w, E, k, C, toks):
    """Dropped assignments contribute nothing (gating.hpp:177-181)."""
    from oracle import native as N

    _, _, dropped = N.ref_static_dispatch(idx, E, C)
    wz = w.copy()
    for t, e in dropped:
        wz[t, int(np.nonzero(idx[t] == e)[0][0])] = 0.0
    return OL.layer_forward(X, W1, W2, idx, wz, E, tokens=toks)


def case_route():
    """moe_route_dynamic / moe_route_static alone, bit-exact vs the reference."""
    import ctypes as C

    from oracle import native as N
    from paper_2303_06182_b200.layer import _stream_ptr

    ctx = Context.get(0)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    rng = np.random.default_rng(7)
    for S, k, E in [(1000, 2, 64), (20000, 2, 512)]:  # one-CTA form, grid form
        ex = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
        d_idx = torch.from_numpy(ex.reshape(-1).copy()).cuda()
        counts = torch.empty(E, dtype=torch.int32, device="cuda")
        pos = torch.empty(S * k, dtype=torch.int32, device="cuda")
        splits = torch.empty(E + 1, dtype=torch.int32, device="cuda")
        order = torch.empty(S * k, dtype=torch.int32, device="cuda")
        assert ctx.lib.moe_route_dynamic(ctx.h, P(d_idx), S, k, E, P(counts), P(splits), P(order), P(pos),
                                         _stream_ptr()) == 0
        assert ctx.lib.moe_check_errors(ctx.h, _stream_ptr()) == 0
        ro, rc, rs = N.ref_dynamic_dispatch(ex, E)
        assert np.array_equal(order.cpu().numpy(), ro) and np.array_equal(splits.cpu().numpy(), rs)
        cap, rslots, rdrop = N.ref_static_dispatch(ex, E, 0.5)
        slots = torch.empty(E * cap, dtype=torch.int32, device="cuda")
        dropped = torch.empty(2 * S * k, dtype=torch.int32, device="cuda")
        nd = torch.zeros(1, dtype=torch.int32, device="cuda")
        assert ctx.lib.moe_route_static(ctx.h, P(d_idx), S, k, E, cap, P(counts), P(slots), P(pos), P(dropped),
                                        P(nd), _stream_ptr()) == 0
        assert ctx.lib.moe_check_errors(ctx.h, _stream_ptr()) == 0
        assert np.array_equal(slots.cpu().numpy().reshape(E, cap), rslots)
        print(f"route S={S} k={k} E={E}: dynamic + static (CF 0.5) bit-exact")


def case_cache():
    S, TD, HD, E, k = 512, 1024, 1024, 32, 2
    shape = LayerShape(TD, HD, E, k)
    Wg, W1, W2 = make_weights(shape)
    W1h, W2h = W1.cpu().pin_memory(), W2.cpu().pin_memory()
    L = MoeLayer(shape, S, weights=(Wg, None, None), pool_only=True)
    cache = ExpertCache(L, 6, W1_host=W1h, W2_host=W2h)
    x = make_tokens(S, TD)
    for _ in range(2):
        out = cache.forward(x)
    torch.cuda.synchronize()
    ref_layer = MoeLayer(shape, S, weights=(Wg, W1, W2))
    ref = ref_layer(x)
    torch.cuda.synchronize()
    assert torch.equal(out, ref), "cache path differs from the resident layer"
    print("cache: bitwise equal to the resident layer;", cache.stats())
    cache.close()
    L.close()
    ref_layer.close()


def case_host():
    S, TD, HD, E, k = 384, 1024, 1024, 16, 2
    shape = LayerShape(TD, HD, E, k)
    W = make_weights(shape)
    L = MoeLayer(shape, S, weights=W)
    xs = [make_tokens(S, TD, seed=11 + i).cpu().pin_memory() for i in range(4)]
    os_ = [torch.empty_like(xs[0]).pin_memory() for _ in range(4)]
    ref = torch.empty_like(xs[0]).pin_memory()
    L.forward_host_batches(xs, os_, torch.cuda.current_stream())
    for i in range(4):
        L.forward_host(xs[i], ref)
        assert torch.equal(ref, os_[i])
    print("host: forward_host_batches == forward_host on 4 batches")
    L.close()


def case_ep1():
    from paper_2303_06182_b200.ep import PeerExpertParallelMoE, Placement

    S, TD, HD, E, k = 512, 1024, 1024, 16, 2
    ctx = Context.get(0)
    shape = LayerShape(TD, HD, E, k)
    Wg, W1, W2 = make_weights(shape, ctx=ctx)
    x = make_tokens(S, TD, ctx=ctx)
    pl = Placement.contiguous(E, 1)
    ep = PeerExpertParallelMoE(ctx, pl, shape, Wg, W1, W2, max_tokens=S, rank=0)
    out = ep.forward(x)
    out = ep.forward(x)
    ep.check_errors()
    torch.cuda.synchronize()
    ref_layer = MoeLayer(shape, S, weights=(Wg, W1, W2))
    ref = ref_layer(x)
    torch.cuda.synchronize()
    assert torch.equal(out, ref), "EP world 1 differs from the single-GPU layer"
    print("ep1: bitwise equal to the single-GPU layer")
    ep.close()
    ref_layer.close()


CASES = {
    "cfg1": lambda: run_layer(512, 1024, 4096, 8, 1),
    "lm": lambda: run_layer(1024, 1024, 1024, 512, 2),
    "mt256": lambda: run_layer(1536, 2048, 2048, 128, 2, tile_n=256),
    "onesm": lambda: (os.environ.__setitem__("MOE_FFN_PAIR", "0"), run_layer(700, 1024, 1024, 64, 2)),
    "split": lambda: run_layer(700, 1024, 1024, 64, 2, split=True),
    "static": lambda: run_layer(640, 1024, 1024, 16, 2, mode="static", C=1.0),
    "graph": lambda: run_layer(512, 1024, 1024, 64, 2, graph=True),
    "route": case_route,
    "cache": case_cache,
    "host": case_host,
    "ep1": case_ep1,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    # a side stream: the graph and pipelined host paths refuse the legacy default stream
    with torch.cuda.stream(torch.cuda.Stream()):
        for n in names:
            CASES[n]()
    torch.cuda.synchronize()
    Context.close_all()  # library allocations end here; what memcheck still lists is torch's pool
    print("OK")
