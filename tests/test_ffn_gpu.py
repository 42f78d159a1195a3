"""GPU tests of the stand-alone grouped FFN (moe_ffn_*, the expert-parallel
receive side), the keyed dispatch and the segment-id helper, each against a
plain fp32 torch reference of the same op."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import layer as OL
from oracle import native as N
from paper_2303_06182_b200 import _capi
from paper_2303_06182_b200.layer import Context, LayerShape, make_weights

pytestmark = pytest.mark.gpu


def P(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def S_():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("R,TD,HD,E,tile_n,with_w", [(700, 256, 512, 8, 128, True), (4096, 1024, 4096, 32, 256, True),
                                                     (4096, 1024, 4096, 32, 128, False), (1, 128, 128, 3, 0, True),
                                                     (5000, 256, 256, 5, 256, True)])
def test_ffn_rows_match_fp32_reference(R, TD, HD, E, tile_n, with_w):
    ctx = Context.get(0)
    shape = LayerShape(TD, HD, E, 1)
    _, W1, W2 = make_weights(shape, seed=11, ctx=ctx)
    g = torch.Generator(device="cuda").manual_seed(R)
    x = (torch.rand(R, TD, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    keys = torch.randint(0, E, (R,), device="cuda", dtype=torch.int32, generator=g)
    w = torch.rand(R, device="cuda", generator=g) if with_w else None
    d = _capi.FfnDesc(R, TD, HD, E, tile_n)
    h = C.c_void_p()
    _capi.check(ctx.lib.moe_ffn_create(ctx.h, C.byref(d), P(W1), P(W2), C.byref(h)))
    y = torch.empty_like(x)
    _capi.check(ctx.lib.moe_ffn_forward(h, P(x), P(keys), P(w), R, P(y), S_()))
    torch.cuda.synchronize()
    ctx.lib.moe_ffn_destroy(h)
    ref = torch.empty(R, TD, device="cuda")
    xf = x.float()
    for e in range(E):
        m = keys == e
        if m.any():
            hh = torch.relu(xf[m] @ W1[e].float().T).bfloat16().float()
            ref[m] = hh @ W2[e].float().T
    if with_w:
        ref *= w[:, None]
    err = OL.rel_fro(y.float().cpu().numpy(), ref.cpu().numpy())
    print(f"ffn R={R} tile_n={tile_n} rel_fro={err:.2e}")
    assert err < 1e-2


def test_route_keyed_matches_oracle():
    ctx = Context.get(0)
    rng = np.random.default_rng(2)
    S, k, E, D = 3000, 2, 64, 4
    idx = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
    dev_of = rng.permutation(np.arange(E) % D).astype(np.int32)
    from paper_2303_06182_b200.ep import Placement

    km = Placement(dev_of, D).key_map()
    w = rng.random((S, k)).astype(np.float32)
    t_idx, t_km, t_w = (torch.from_numpy(a).cuda() for a in (idx, km, w))
    counts = torch.empty(E, dtype=torch.int32, device="cuda")
    splits = torch.empty(E + 1, dtype=torch.int32, device="cuda")
    order = torch.empty(S * k, dtype=torch.int32, device="cuda")
    pos = torch.empty(S * k, dtype=torch.int32, device="cuda")
    wpos = torch.empty(S * k, dtype=torch.float32, device="cuda")
    _capi.check(ctx.lib.moe_route_dynamic_keyed(ctx.h, P(t_idx), S, k, E, P(t_km), E, P(counts), P(splits),
                                                P(order), P(pos), P(t_w), P(wpos), S_()))
    _capi.check(ctx.lib.moe_check_errors(ctx.h, S_()))
    o, c, s, p = N.c_dynamic_dispatch(km[idx], E)
    assert (order.cpu().numpy() == o).all() and (counts.cpu().numpy() == c).all()
    assert (pos.cpu().numpy() == p).all()
    assert (wpos.cpu().numpy() == w.reshape(-1)[o]).all()


def test_fill_segments():
    ctx = Context.get(0)
    counts = torch.tensor([3, 0, 5, 1, 0, 2], dtype=torch.int32, device="cuda")
    out = torch.full((11,), -1, dtype=torch.int32, device="cuda")
    _capi.check(ctx.lib.moe_fill_segments(ctx.h, P(counts), 6, 3, P(out), S_()))
    torch.cuda.synchronize()
    assert out.cpu().tolist() == [0, 0, 0, 2, 2, 2, 2, 2, 0, 2, 2]
