"""Expert buffering on the GPU: cache decisions equal the reference's
access_batch (buffer.cpp:57-130, verbatim build) batch by batch, and the
cached layer's outputs are bitwise those of the fully resident layer."""
import numpy as np
import pytest
import torch

from oracle import native as N
from paper_2303_06182_b200.layer import ExpertCache, LayerShape, MoeLayer, make_tokens, make_weights
from paper_2303_06182_b200.traces import skewed_routing

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("policy,slots,frac,pers", [("lifo", 5, 0.5, 0.5), ("fifo", 5, 0.5, 0.5),
                                                    ("lifo", 3, 1.0, 0.9), ("lifo", 16, 1.0, 0.0)])
def test_cache_matches_reference_decisions_and_resident_layer(policy, slots, frac, pers):
    S, TD, HD, E, k, B = 512, 256, 512, 16, 2, 8
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=3)
    full = MoeLayer(shape, S, weights=w)
    cached_layer = MoeLayer(shape, S, weights=w)
    cache = ExpertCache(cached_layer, slots, policy)
    x = make_tokens(S, TD, seed=4)
    ex, wt = skewed_routing(E, k, B, S, 1.2, pers, frac, seed=17)
    ref = N.RefCache()
    pol = {"lifo": 0, "fifo": 1}[policy]
    for b in range(B):
        idx = torch.from_numpy(ex[b]).cuda()
        gw = torch.from_numpy(wt[b].astype(np.float32)).cuda()
        out_c = cache.forward_routed(x, idx, gw)
        out_f = full.forward_routed(x, idx, gw)
        torch.cuda.synchronize()
        assert torch.equal(out_c, out_f), f"batch {b}: cached output differs"
        active = np.unique(ex[b])
        stats, resident = ref.access(active, slots, pol)
        st = cache.stats()["last"]
        assert (st["accesses"], st["hits"], st["misses"], st["evictions"]) == stats, b
        assert cache.resident() == resident, b
    cache.close()


@pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("policy,slots", [("lifo", 4), ("fifo", 6)])
def test_pool_only_cached_layer_holds_only_the_slots(policy, slots):
    """A pool-only layer (no W1/W2 on the device, no packed copy): the cache's
    slot pool is the only expert memory, decisions still equal access_batch,
    outputs still bitwise those of the resident layer (per-slot copy readiness
    included), and a forward without an attached cache is refused."""
    from paper_2303_06182_b200._capi import MoeError

    S, TD, HD, E, k, B = 512, 256, 1024, 32, 2, 10
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=5)
    full = MoeLayer(shape, S, weights=w)
    W1h, W2h = w[1].cpu().pin_memory(), w[2].cpu().pin_memory()
    x = make_tokens(S, TD, seed=6)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    bare = MoeLayer(shape, S, weights=(w[0], None, None), pool_only=True)
    torch.cuda.synchronize()
    layer_bytes = free0 - torch.cuda.mem_get_info()[0]
    expert_bytes = E * 2 * TD * HD * 2
    assert layer_bytes < expert_bytes // 4, (layer_bytes, expert_bytes)
    with pytest.raises(MoeError, match="no expert weights"):
        bare(x)
        torch.cuda.synchronize()
    cache = ExpertCache(bare, slots, policy, W1h, W2h)
    ex, wt = skewed_routing(E, k, B, S, 1.0, 0.3, 0.8, seed=23)
    ref = N.RefCache()
    for b in range(B):
        idx = torch.from_numpy(ex[b]).cuda()
        gw = torch.from_numpy(wt[b].astype(np.float32)).cuda()
        out_c = cache.forward_routed(x, idx, gw)
        out_f = full.forward_routed(x, idx, gw)
        torch.cuda.synchronize()
        assert torch.equal(out_c, out_f), f"batch {b}"
        stats, resident = ref.access(np.unique(ex[b]), slots, {"lifo": 0, "fifo": 1}[policy])
        st = cache.stats()["last"]
        assert (st["accesses"], st["hits"], st["misses"], st["evictions"]) == stats, b
        assert cache.resident() == resident, b
    # the gated forward through the cache works as well
    out_g = cache.forward(x)
    torch.cuda.synchronize()
    assert torch.equal(out_g, full(x))
    cache.close()
