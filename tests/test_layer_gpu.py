"""GPU parity of the MoE layer: gate (logits + top-k), dispatch, gather, grouped
FFN, combine -- each stage against the CPU oracle / a plain fp32 reference.

Tiers (north_star):
  * routing: bit-exact given the same logits -- top-k of the GPU's own fp32
    logits recomputed by the oracle must equal the GPU's idx; dispatch of that
    idx by the C restatement must equal the GPU's order/counts/splits.
  * outputs: within tolerance of an fp32 oracle run with the GPU's routing:
      relative Frobenius error <= 1e-2 (bf16 weights/activations, fp32
      accumulate, bf16 H and output), stated per test below.
"""
import math
import os

import numpy as np
import pytest
import torch

from oracle import layer as OL
from oracle import native as N
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights

pytestmark = pytest.mark.gpu
SEED = 2303061820
TOL_OUT = 1e-2     # rel. Frobenius, layer output vs fp32 oracle (same routing)
TOL_STAGE = 1e-2   # rel. Frobenius, H / Yw vs fp32 reference of the stage


def _f32(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def _run(S, TD, HD, E, k, mode="dynamic", C=1.0, tile_n=0, weights=None, x=None):
    shape = LayerShape(TD, HD, E, k)
    w = weights or make_weights(shape, seed=SEED)
    # split_ffn: the stage checks read H, which the fused FFN drops from L2
    layer = MoeLayer(shape, S, mode=mode, capacity_factor=C, weights=w, keep_logits=True, tile_n=tile_n,
                     split_ffn=True)
    x = make_tokens(S, TD, seed=SEED) if x is None else x
    out = layer(x)
    torch.cuda.synchronize()
    layer.check_errors()
    return layer, x, out, w, layer.view()


def test_synthetic_generator_bit_exact_vs_oracle():
    x = make_tokens(1000, 256, seed=SEED)
    ref = OL.synth_bf16((1000, 256), SEED, OL.T_X, math.sqrt(3.0))
    assert (x.view(torch.int16).cpu().numpy().view(np.uint16) == ref).all()
    shape = LayerShape(128, 256, 4, 1)
    Wg, W1, W2 = make_weights(shape, seed=SEED)
    s = OL.init_scales(128, 256)
    assert (W1.view(torch.int16).cpu().numpy().view(np.uint16) ==
            OL.synth_bf16((4, 256, 128), SEED, OL.T_W1, s["w1"])).all()
    assert (W2.view(torch.int16).cpu().numpy().view(np.uint16) ==
            OL.synth_bf16((4, 128, 256), SEED, OL.T_W2, s["w2"])).all()
    assert (Wg.view(torch.int16).cpu().numpy().view(np.uint16) ==
            OL.synth_bf16((4, 128), SEED, OL.T_WG, s["wg"])).all()


def _check_routing(layer, x, w, v, S, E, k):
    X = _f32(x)
    Wg = _f32(w[0])
    logits = v["logits"][:S * E].reshape(S, E).cpu().numpy()
    ref_logits = OL.gate_logits(X, Wg)
    scale = np.abs(ref_logits).max()
    assert np.abs(logits - ref_logits).max() <= 2e-5 * max(scale, 1.0) * math.sqrt(X.shape[1] / 256)
    # routing tier: bit-exact given the GPU's logits
    idx = v["idx"][:S * k].reshape(S, k).cpu().numpy()
    ridx, rw = OL.topk_from_logits(logits, k)
    assert (idx == ridx).all()
    gw = v["w"][:S * k].reshape(S, k).cpu().numpy()
    assert np.abs(gw - rw).max() < 2e-6
    assert np.abs(gw.astype(np.float64).sum(1) - 1.0).max() < 1e-6
    return idx, gw


@pytest.mark.parametrize("S,TD,HD,E,k,tile_n", [(300, 256, 512, 8, 2, 0), (1000, 256, 384, 16, 1, 0),
                                                (257, 128, 256, 33, 3, 256), (64, 512, 256, 512, 2, 0),
                                                # k = 4 (per-k gather/combine), k = 6 (generic row
                                                # forms), TD = 1152 (a 4-vector sweep plus a tail)
                                                (333, 128, 256, 12, 4, 0), (200, 256, 256, 40, 6, 0),
                                                (129, 1152, 256, 9, 4, 0)])
def test_layer_small_all_stages(S, TD, HD, E, k, tile_n):
    layer, x, out, w, v = _run(S, TD, HD, E, k, tile_n=tile_n)
    idx, gw = _check_routing(layer, x, w, v, S, E, k)
    order, counts, splits, pos = N.c_dynamic_dispatch(idx, E)
    assert (v["order"].cpu().numpy()[:S * k] == order).all()
    assert (v["counts"].cpu().numpy() == counts).all()
    assert (v["splits"].cpu().numpy() == splits).all()
    assert (v["pos"].cpu().numpy()[:S * k] == pos).all()
    # gather: bitwise
    xp = v["xp"].view(S * k, TD)
    assert torch.equal(xp, x[torch.from_numpy(order // k).long().cuda()])
    # grouped FFN stage by stage vs fp32 torch reference of the same op
    W1 = w[1].float()
    W2 = w[2].float()
    h = v["h"].view(S * k, HD).float()
    yw = v["yw"].view(S * k, TD).float()
    h_ref = torch.empty_like(h)
    y_ref = torch.empty_like(yw)
    wpos = torch.from_numpy(gw.reshape(-1)[order]).cuda()
    for e in range(E):
        a, b = int(splits[e]), int(splits[e + 1])
        if a == b:
            continue
        h_ref[a:b] = torch.relu(xp[a:b].float() @ W1[e].T)
        y_ref[a:b] = (h[a:b] @ W2[e].T) * wpos[a:b, None]
    assert OL.rel_fro(h.cpu().numpy(), h_ref.cpu().numpy()) < TOL_STAGE
    assert OL.rel_fro(yw.cpu().numpy(), y_ref.cpu().numpy()) < TOL_STAGE
    # whole layer vs the numpy oracle with the GPU's routing
    ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), idx, gw.astype(np.float64), E)
    err = OL.rel_fro(_f32(out), ref)
    print(f"layer rel_fro={err:.2e}")
    assert err < TOL_OUT


@pytest.mark.parametrize("S,TD,E,k", [(130, 128, 8, 2),     # small-E CUDA-core gate
                                      (300, 256, 512, 2),   # tcgen05 gate, 2 x N=256 MMAs, 32-deep
                                      (300, 256, 512, 4),
                                      (260, 256, 200, 3),   # tcgen05 gate, one N=208 MMA
                                      (200, 256, 96, 2)])   # 64-deep tcgen05 gate
def test_gate_ties_go_to_lower_expert(S, TD, E, k):
    HD = 128
    shape = LayerShape(TD, HD, E, k)
    Wg, W1, W2 = make_weights(shape, seed=SEED)
    Wg[:] = Wg[0:1]  # every expert row identical -> all logits equal
    layer, x, out, w, v = _run(S, TD, HD, E, k, weights=(Wg, W1, W2))
    idx = v["idx"][:S * k].reshape(S, k).cpu().numpy()
    assert (idx == np.arange(k)).all()
    assert np.allclose(v["w"][:S * k].cpu().numpy(), 1.0 / k)


def test_layer_cfg1_shape():
    """configs[0] shape: TD=1024 HD=4096 E=8 top-1, 2048 tokens (tile_n auto =
    128: 256 rows per expert, but 256-token items would leave only ~2 waves of
    tiles for 8 experts), and the 256-token items forced."""
    S, TD, HD, E, k = 2048, 1024, 4096, 8, 1
    layer, x, out, w, v = _run(S, TD, HD, E, k)
    assert v["tile_n"] == 128
    layer256, _, out256, _, v256 = _run(S, TD, HD, E, k, tile_n=256, weights=w, x=x)
    assert v256["tile_n"] == 256
    assert torch.equal(out, out256)  # a row's FFN does not depend on the item width
    idx, gw = _check_routing(layer, x, w, v, S, E, k)
    order, counts, splits, pos = N.c_dynamic_dispatch(idx, E)
    assert (v["order"].cpu().numpy()[:S * k] == order).all()
    # full-layer fp32 torch reference on the GPU (same routing)
    xf, W1, W2 = x.float(), w[1].float(), w[2].float()
    ref = torch.zeros(S, TD, device="cuda")
    it = torch.from_numpy(idx).long().cuda()
    wt = torch.from_numpy(gw).cuda()
    for e in range(E):
        for j in range(k):
            m = it[:, j] == e
            if m.any():
                ref[m] += wt[m, j:j + 1] * (torch.relu(xf[m] @ W1[e].T) @ W2[e].T)
    err = OL.rel_fro(_f32(out), ref.cpu().numpy())
    print(f"cfg1 rel_fro={err:.2e}")
    assert err < TOL_OUT
    # and the numpy oracle on a token subset
    toks = np.arange(0, S, 97)
    o = OL.layer_forward(_f32(x), lambda e: _f32(w[1][e]), lambda e: _f32(w[2][e]), idx,
                         gw.astype(np.float64), E, tokens=toks)
    assert OL.rel_fro(_f32(out)[toks], o) < TOL_OUT


def test_layer_cfg2_shape_subset():
    """configs[1] shape: LM TD=1024 HD=4096 E=512 k=2, 8x2048 tokens."""
    S, TD, HD, E, k = 16384, 1024, 4096, 512, 2
    layer, x, out, w, v = _run(S, TD, HD, E, k)
    idx, gw = _check_routing(layer, x, w, v, S, E, k)
    order, counts, splits, pos = N.c_dynamic_dispatch(idx, E)
    assert (v["order"].cpu().numpy()[:S * k] == order).all()
    assert (v["counts"].cpu().numpy() == counts).all()
    toks = np.arange(3, S, 1021)
    xf = x.float()
    ref = torch.zeros(len(toks), TD, device="cuda")
    for r, t in enumerate(toks):
        for j in range(k):
            e = int(idx[t, j])
            hh = torch.relu(xf[t] @ w[1][e].float().T)
            ref[r] += float(gw[t, j]) * (hh @ w[2][e].float().T)
    err = OL.rel_fro(_f32(out)[toks], ref.cpu().numpy())
    print(f"cfg2 subset rel_fro={err:.2e}")
    assert err < TOL_OUT


@pytest.mark.parametrize("S,TD,HD,E,k,C", [(512, 256, 256, 8, 2, 0.3), (300, 128, 256, 4, 1, 1.0),
                                           (2048, 256, 256, 64, 2, 0.05)])
def test_static_mode_matches_oracle(S, TD, HD, E, k, C):
    layer, x, out, w, v = _run(S, TD, HD, E, k, mode="static", C=C)
    idx = v["idx"][:S * k].reshape(S, k).cpu().numpy()
    gw = v["w"][:S * k].reshape(S, k).cpu().numpy()
    cap, slots, dropped, pos = N.c_static_dispatch(idx, E, C)
    assert v["capacity"] == cap
    assert (v["order"].cpu().numpy()[:E * cap].reshape(E, cap) == slots).all()
    nd = int(v["n_dropped"].item())
    assert nd == len(dropped)
    assert (v["dropped"].cpu().numpy()[:2 * nd].reshape(-1, 2) == dropped).all()
    assert (v["pos"].cpu().numpy()[:S * k] == pos).all()
    # oracle: dropped assignments contribute nothing (gating.hpp:177-181)
    wz = gw.astype(np.float64).copy()
    wz.reshape(-1)[pos < 0] = 0.0
    ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), idx, wz, E)
    err = OL.rel_fro(_f32(out), ref)
    print(f"static rel_fro={err:.2e} dropped={nd}")
    assert err < TOL_OUT


@pytest.mark.parametrize("S,TD,HD,E,k", [(1024, 256, 512, 16, 2), (16384, 1024, 4096, 512, 2)])
def test_graph_and_host_paths_bitwise_equal_to_eager(S, TD, HD, E, k):
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    layer = MoeLayer(shape, S, weights=w)
    x = make_tokens(S, TD, seed=SEED)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
    with torch.cuda.stream(s):
        eager = layer(x, stream=s)
        out_g = torch.empty_like(x)
        layer.forward(x, out_g, graph=True, stream=s)
        layer.forward(x, out_g, graph=True, stream=s)  # replay
    s.synchronize()
    assert torch.equal(eager, out_g)
    xh = x.cpu().pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    layer.forward_host(xh, oh, stream=s)
    assert torch.equal(oh, eager.cpu())


@pytest.mark.parametrize("S,TD,HD,E,k", [(1024, 256, 512, 16, 2), (16384, 1024, 4096, 512, 2)])
def test_pipelined_host_batches_bitwise_equal_per_call(S, TD, HD, E, k):
    """moe_layer_forward_host_batches: every batch of the queue (different
    tokens, different sizes, triple-buffered staging reused) equals its own
    synchronous moe_layer_forward_host call."""
    shape = LayerShape(TD, HD, E, k)
    layer = MoeLayer(shape, S, weights=make_weights(shape, seed=SEED))
    sizes = [S, S // 2 + 3, S, 1, S - 7, S]
    xs = [make_tokens(n, TD, seed=SEED + 10 + i).cpu().pin_memory() for i, n in enumerate(sizes)]
    outs = [torch.empty_like(x).pin_memory() for x in xs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # inputs were written on the current stream
    layer.forward_host_batches(xs, outs, s)
    for x, o in zip(xs, outs):
        ref = torch.empty_like(x).pin_memory()
        layer.forward_host(x, ref, stream=s)
        assert torch.equal(o, ref)
    # outputs written to a shared ring of buffers stay ordered
    ring = [torch.empty_like(xs[0]).pin_memory() for _ in range(2)]
    layer.forward_host_batches([xs[0], xs[2], xs[0], xs[2], xs[0]], [ring[0], ring[1]] * 2 + [ring[0]], s)
    assert torch.equal(ring[0], outs[0]) and torch.equal(ring[1], outs[2])


@pytest.mark.parametrize("S,TD,HD,E,k", [(1024, 256, 512, 16, 2), (16384, 1024, 4096, 512, 2)])
def test_packed_weights_bitwise_equal_row_major_and_repack(S, TD, HD, E, k):
    """The fused FFN's prepacked weight copy (default) gives the same bits as
    streaming the caller's row-major weights (keep_layout), and
    moe_layer_repack picks up in-place weight updates."""
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    x = make_tokens(S, TD, seed=SEED)
    packed = MoeLayer(shape, S, weights=w)
    plain = MoeLayer(shape, S, weights=w, keep_layout=True)
    a, b = packed(x), plain(x)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    w[1].mul_(-1.0)  # in place: the packed copy is stale until repack
    torch.cuda.synchronize()
    packed.repack()
    a2, b2 = packed(x), plain(x)
    torch.cuda.synchronize()
    assert torch.equal(a2, b2) and not torch.equal(a2, a)


def test_repeat_forward_is_deterministic():
    layer, x, out, w, v = _run(4096, 256, 512, 64, 2)
    out2 = layer(x)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)


@pytest.mark.parametrize("S,TD,HD,E,k", [(1000, 256, 384, 16, 1), (2048, 1024, 4096, 8, 1),
                                         (4096, 1024, 2048, 64, 1), (16384, 1024, 4096, 512, 1)])
@pytest.mark.parametrize("split", [False, True])
def test_top1_direct_store_bitwise_equal_combine_kernel(S, TD, HD, E, k, split):
    """fuse_combine on a top-1 layer: GEMM2 writes each token's output row
    itself (in the persistent fused FFN -- 1-SM or CTA-pair kernel -- and in
    the two-launch grouped GEMM); bitwise the combine kernel's result."""
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    x = make_tokens(S, TD, seed=SEED)
    fused = MoeLayer(shape, S, weights=w, fuse_combine=True, split_ffn=split)
    plain = MoeLayer(shape, S, weights=w, split_ffn=split)
    a = fused(x)
    b = plain(x)
    a2 = fused(x)
    torch.cuda.synchronize()
    fused.check_errors()
    assert torch.equal(a, b)
    assert torch.equal(a, a2)


def test_fuse_combine_refused_for_top2():
    from paper_2303_06182_b200._capi import MoeError

    shape = LayerShape(256, 256, 8, 2)
    with pytest.raises(MoeError, match="top-1"):
        MoeLayer(shape, 64, weights=make_weights(shape, seed=SEED), fuse_combine=True)


@pytest.mark.parametrize("S,TD,HD,E,k,mode,C", [(300, 256, 512, 8, 2, "dynamic", 1.0), (2048, 1024, 4096, 8, 1, "dynamic", 1.0),
                                                (257, 128, 256, 33, 3, "dynamic", 1.0),
                                                (16384, 1024, 4096, 512, 2, "dynamic", 1.0),
                                                (512, 256, 256, 8, 2, "static", 0.3), (6144, 2048, 8192, 128, 2, "dynamic", 1.0)])
def test_fused_ffn_bitwise_equal_two_launch_ffn(S, TD, HD, E, k, mode, C):
    """One persistent launch with H kept in L2 (ffn_fused.cu) == GEMM1 and GEMM2
    as two launches: same tiles, same K order, same epilogues."""
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    x = make_tokens(S, TD, seed=SEED)
    fused = MoeLayer(shape, S, weights=w, mode=mode, capacity_factor=C)
    split = MoeLayer(shape, S, weights=w, mode=mode, capacity_factor=C, split_ffn=True)
    a = fused(x)
    b = split(x)
    a2 = fused(x)
    torch.cuda.synchronize()
    fused.check_errors()
    assert torch.equal(a, b)
    assert torch.equal(a, a2)


_GATE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights
S, TD, HD, E, k = map(int, sys.argv[2:7])
shape = LayerShape(TD, HD, E, k)
layer = MoeLayer(shape, S, weights=make_weights(shape, seed=2303061820), keep_logits=True)
layer(make_tokens(S, TD, seed=2303061820))
torch.cuda.synchronize()
np.save(sys.argv[7], layer.view()["logits"][:S * E].cpu().numpy())
np.save(sys.argv[7] + ".idx.npy", layer.view()["idx"][:S * k].cpu().numpy())
"""


@pytest.mark.parametrize("S,TD,HD,E,k", [(2048, 1024, 4096, 8, 1), (300, 256, 512, 9, 2),
                                         (1000, 512, 512, 32, 4), (129, 1152, 256, 16, 2)])
def test_small_e_gate_matches_tcgen05_gate(S, TD, HD, E, k, tmp_path):
    """E <= 32: the CUDA-core gate (gate_small_kernel) against the tcgen05
    gate (MOE_GATE_SMALL=0, a separate process since the choice is read once):
    both within the fp32 oracle's tolerance, and each one's routing equal to
    the top-k of its own logits."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for small in ("1", "0"):
        f = str(tmp_path / f"logits_{small}.npy")
        env = dict(os.environ, MOE_GATE_SMALL=small)
        r = subprocess.run([sys.executable, "-c", _GATE_SCRIPT, root, str(S), str(TD), str(HD), str(E), str(k), f],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[small] = np.load(f).reshape(S, E)
        idx = np.load(f + ".idx.npy").reshape(S, k)
        assert (idx == OL.topk_from_logits(outs[small], k)[0]).all(), small
    x = _f32(make_tokens(S, TD, seed=SEED))
    Wg = _f32(make_weights(LayerShape(TD, HD, E, k), seed=SEED)[0])
    ref = OL.gate_logits(x, Wg)
    tol = 2e-5 * max(float(np.abs(ref).max()), 1.0) * math.sqrt(TD / 256)
    for small, lg in outs.items():
        assert np.abs(lg - ref).max() <= tol, small
    assert np.abs(outs["1"] - outs["0"]).max() <= tol


@pytest.mark.parametrize("S,TD,HD,E,k", [(2048, 1024, 4096, 8, 1), (6144, 2048, 8192, 128, 2),
                                         (300, 256, 512, 40, 2)])
def test_split_k_gate_matches_one_cta_gate(S, TD, HD, E, k, tmp_path):
    """The split-K gate (a cluster of CTAs per token tile, partial logits
    reduced over DSMEM: MT, cfg1 and small batches) against the one-CTA-per-
    tile gate (MOE_GATE_SPLIT=0, a separate process since the choice is read
    once): same logits up to fp32 summation order, both checked against the
    fp32 oracle."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for split in ("8", "0"):
        f = str(tmp_path / f"logits_{split}.npy")
        env = dict(os.environ, MOE_GATE_SPLIT=split)
        r = subprocess.run([sys.executable, "-c", _GATE_SCRIPT, root, str(S), str(TD), str(HD), str(E), str(k), f],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[split] = np.load(f).reshape(S, E)
    x = _f32(make_tokens(S, TD, seed=SEED))
    Wg = _f32(make_weights(LayerShape(TD, HD, E, k), seed=SEED)[0])
    ref = OL.gate_logits(x, Wg)
    tol = 2e-5 * max(float(np.abs(ref).max()), 1.0) * math.sqrt(TD / 256)
    for split, lg in outs.items():
        assert np.abs(lg - ref).max() <= tol, split
    assert np.abs(outs["8"] - outs["0"]).max() <= tol


@pytest.mark.parametrize("S,TD,HD,E,k,mode,C", [
    (1, 256, 256, 16, 2, "dynamic", 1.0),      # a single token
    (127, 128, 256, 8, 8, "dynamic", 1.0),     # k == E: every expert gets every token
    (129, 256, 512, 5, 1, "dynamic", 1.0),     # E not a power of two, S not a tile multiple
    (4097, 256, 256, 64, 2, "dynamic", 1.0),   # just past the single-CTA route (multi-block sort)
    (300, 256, 512, 8, 2, "static", 0.1),      # static with drops, one-launch fused FFN
    (1, 256, 256, 512, 2, "dynamic", 1.0),     # a single token through the E = 512 tcgen05 gate
    (3, 256, 256, 1, 1, "dynamic", 1.0),       # one expert
    (33, 256, 256, 33, 2, "dynamic", 1.0),     # first E past the CUDA-core gate (64-deep, E_pad 48)
    (200, 256, 256, 128, 8, "dynamic", 1.0),   # k = 8 on the tcgen05 gate
])
def test_layer_edge_shapes_fused_default(S, TD, HD, E, k, mode, C):
    """The default (fused, packed) path on edge shapes: routing bit-exact,
    output within TOL_OUT of the fp32 oracle run with the GPU's routing."""
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    layer = MoeLayer(shape, S, mode=mode, capacity_factor=C, weights=w, keep_logits=True)
    x = make_tokens(S, TD, seed=SEED)
    out = layer(x)
    torch.cuda.synchronize()
    layer.check_errors()
    v = layer.view()
    idx, gw = _check_routing(layer, x, w, v, S, E, k)
    if mode == "dynamic":
        ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), idx, gw.astype(np.float64), E)
    else:
        cap, slots, dropped, pos = N.c_static_dispatch(idx, E, C)
        assert (v["order"].cpu().numpy()[:E * cap].reshape(E, cap) == slots).all()
        wz = gw.astype(np.float64).copy()
        wz.reshape(-1)[pos < 0] = 0.0  # dropped assignments contribute nothing (gating.hpp:177-181)
        ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), idx, wz, E)
    err = OL.rel_fro(_f32(out), ref)
    print(f"{mode} S={S} E={E} k={k}: rel_fro={err:.2e}")
    assert err < TOL_OUT


@pytest.mark.parametrize("k", [1, 2])
def test_layer_routed_all_tokens_on_few_experts(k):
    """Caller routing that puts every token on expert 3 (and 5): S rows on one
    expert (many work items of one expert), every other expert empty."""
    S, TD, HD, E = 1000, 256, 512, 16
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    layer = MoeLayer(shape, S, weights=w)
    x = make_tokens(S, TD, seed=SEED)
    ex = np.tile(np.array([3, 5][:k], np.int32), (S, 1))
    gw = np.tile(np.array([0.75, 0.25][:k] if k == 2 else [1.0], np.float32), (S, 1))
    out = layer.forward_routed(x, torch.from_numpy(ex).cuda(), torch.from_numpy(gw).cuda())
    torch.cuda.synchronize()
    layer.check_errors()
    v = layer.view()
    counts = v["counts"].cpu().numpy()
    assert counts[3] == S and counts.sum() == S * k
    ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), ex, gw.astype(np.float64), E)
    err = OL.rel_fro(_f32(out), ref)
    assert err < TOL_OUT


def test_invalid_expert_ids_fail_cleanly_and_layer_recovers():
    """Caller routing with ids outside [0, E) on a fresh layer: the forward
    reports the reference's range error (no stale row indices reach the
    gather, no device fault), and the next valid forward is exact."""
    from paper_2303_06182_b200._capi import MoeError

    S, TD, HD, E, k = 300, 256, 512, 8, 2
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    layer = MoeLayer(shape, S, weights=w)
    x = make_tokens(S, TD, seed=SEED)
    rng = np.random.default_rng(7)
    ex = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
    gw = np.full((S, k), 0.5, np.float32)
    bad = ex.copy()
    bad[7, 1] = E
    bad[100, 0] = -1
    with pytest.raises(MoeError):
        layer.forward_routed(x, torch.from_numpy(bad).cuda(), torch.from_numpy(gw).cuda())
        torch.cuda.synchronize()
        layer.check_errors()
    out = layer.forward_routed(x, torch.from_numpy(ex).cuda(), torch.from_numpy(gw).cuda())
    torch.cuda.synchronize()
    layer.check_errors()
    ref = OL.layer_forward(_f32(x), _f32(w[1]), _f32(w[2]), ex, gw.astype(np.float64), E)
    assert OL.rel_fro(_f32(out), ref) < TOL_OUT


@pytest.mark.parametrize("S,TD,HD,E,k", [(1024, 256, 512, 16, 2), (2048, 1024, 4096, 8, 1),
                                         (16384, 1024, 4096, 512, 2), (12288, 2048, 8192, 128, 2)])
def test_pack_in_place_holds_expert_weights_once(S, TD, HD, E, k):
    """moe_pack_expert_weights in place + weights_packed: the layer streams the
    caller's (repacked) buffers and allocates no expert-weight copy; outputs
    bitwise equal to the default layer (which streams its own packed copy)."""
    shape = LayerShape(TD, HD, E, k)
    x = make_tokens(S, TD, seed=SEED)
    ref_layer = MoeLayer(shape, S, weights=make_weights(shape, seed=SEED))
    ref = ref_layer(x)
    torch.cuda.synchronize()
    ref_layer.close()
    del ref_layer
    torch.cuda.empty_cache()
    w = make_weights(shape, seed=SEED)

    def allocated_by(make):
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        obj = make()
        torch.cuda.synchronize()
        return obj, free0 - torch.cuda.mem_get_info()[0]

    copy_layer, extra_copy = allocated_by(lambda: MoeLayer(shape, S, weights=w))
    copy_layer.close()
    del copy_layer
    torch.cuda.empty_cache()
    layer, extra = allocated_by(lambda: MoeLayer(shape, S, weights=w, pack_in_place=True))
    expert_bytes = E * 2 * TD * HD * 2
    print(f"layer allocations {extra / 1e6:.1f} MB (default layer {extra_copy / 1e6:.1f} MB) "
          f"for {expert_bytes / 1e6:.1f} MB of experts")
    assert extra_copy - extra >= 0.9 * expert_bytes
    out = layer(x)
    out2 = layer(x)
    torch.cuda.synchronize()
    layer.check_errors()
    assert torch.equal(out, ref) and torch.equal(out2, ref)
    assert layer.view()["ffn_kernel"] in (1, 2)


_OUT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights
S, TD, HD, E, k = map(int, sys.argv[2:7])
shape = LayerShape(TD, HD, E, k)
layer = MoeLayer(shape, S, weights=make_weights(shape, seed=2303061820))
x = make_tokens(S, TD, seed=2303061820)
for _ in range(3):  # repeated forwards: dirty / discarded H lines of the previous step
    out = layer(x)
torch.cuda.synchronize()
layer.check_errors()
np.save(sys.argv[7], out.float().cpu().numpy())
"""


@pytest.mark.parametrize("S,TD,HD,E,k", [(2048, 1024, 4096, 8, 1), (4096, 512, 1024, 64, 2)])
def test_h_discard_does_not_change_outputs(S, TD, HD, E, k, tmp_path):
    """The fused FFN drops consumed H lines from L2 only when H exceeds half of
    L2 (capi.cu ffn_discard_h); forcing the discard on and off (separate
    processes: MOE_FFN_DISCARD is read once) must give bitwise-equal layer
    outputs over repeated forwards."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for d in ("1", "0"):
        f = str(tmp_path / f"out_{d}.npy")
        env = dict(os.environ, MOE_FFN_DISCARD=d)
        r = subprocess.run([sys.executable, "-c", _OUT_SCRIPT, root, str(S), str(TD), str(HD), str(E), str(k), f],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[d] = np.load(f)
    assert np.array_equal(outs["1"], outs["0"])
    assert np.isfinite(outs["0"]).all() and np.abs(outs["0"]).max() > 0


@pytest.mark.parametrize("S,TD,HD,E,k", [(8192, 1024, 4096, 128, 2), (2048, 1024, 4096, 8, 1)])
def test_ffn_schedule_does_not_change_outputs(S, TD, HD, E, k, tmp_path):
    """Which CTA (pair) runs a tile is a scheduling choice: the round-robin body,
    the dynamically claimed tail (default: >= 7 waves of pair-tiles in the
    CTA-pair kernel) and an all-dynamic schedule must give bitwise-equal layer
    outputs (MOE_FFN_DYN_TAIL is read once: separate processes).  The first
    shape runs the CTA-pair kernel, the second (configs[0]) the 1-SM kernel."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for t in ("0", "2", "100000"):
        f = str(tmp_path / f"out_{t}.npy")
        env = dict(os.environ, MOE_FFN_DYN_TAIL=t)
        r = subprocess.run([sys.executable, "-c", _OUT_SCRIPT, root, str(S), str(TD), str(HD), str(E), str(k), f],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[t] = np.load(f)
    assert np.array_equal(outs["0"], outs["2"])
    assert np.array_equal(outs["0"], outs["100000"])
    assert np.isfinite(outs["0"]).all() and np.abs(outs["0"]).max() > 0
