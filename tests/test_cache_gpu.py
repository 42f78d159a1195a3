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
