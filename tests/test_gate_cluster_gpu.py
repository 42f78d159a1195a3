"""Gate with Wg multicast across a CTA cluster (gate.cu): routing parity vs the
oracle for expert counts that use 1-, 2- and 4-CTA clusters and token counts
that leave idle CTAs in the last cluster; logits/idx/w bitwise independent of
the cluster size (MOE_GATE_CLUSTER, read once per process -> subprocesses)."""
import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import layer as OL
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights

pytestmark = pytest.mark.gpu
SEED = 2303061820
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gate(S, TD, E, k):
    shape = LayerShape(TD, 256, E, k)
    w = make_weights(shape, seed=SEED)
    layer = MoeLayer(shape, S, weights=w, keep_logits=True)
    x = make_tokens(S, TD, seed=SEED)
    layer(x)
    torch.cuda.synchronize()
    layer.check_errors()
    v = layer.view()
    return x, w, v


@pytest.mark.parametrize("S,TD,E,k", [(1300, 256, 128, 2), (1000, 512, 160, 2), (517, 256, 272, 1),
                                      (4100, 1024, 512, 2), (640, 256, 496, 4)])
def test_gate_cluster_routing_matches_oracle(S, TD, E, k):
    x, w, v = _gate(S, TD, E, k)
    X = x.float().cpu().numpy()
    logits = v["logits"][:S * E].reshape(S, E).cpu().numpy()
    ref = OL.gate_logits(X, w[0].float().cpu().numpy())
    assert np.abs(logits - ref).max() <= 2e-5 * max(np.abs(ref).max(), 1.0) * np.sqrt(TD / 256)
    idx = v["idx"][:S * k].reshape(S, k).cpu().numpy()
    ridx, rw = OL.topk_from_logits(logits, k)
    assert (idx == ridx).all()
    assert np.abs(v["w"][:S * k].reshape(S, k).cpu().numpy() - rw).max() < 2e-6


_SCRIPT = r"""
import hashlib, sys, torch
sys.path.insert(0, %r)
from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights
out = []
for S, TD, E, k in [(16384, 1024, 512, 2), (1300, 256, 160, 2)]:
    shape = LayerShape(TD, 256, E, k)
    layer = MoeLayer(shape, S, weights=make_weights(shape, seed=7), keep_logits=True)
    layer(make_tokens(S, TD, seed=7))
    torch.cuda.synchronize()
    layer.check_errors()
    v = layer.view()
    h = hashlib.sha256()
    for name, n in (("logits", S * E), ("idx", S * k), ("w", S * k)):
        h.update(v[name][:n].cpu().numpy().tobytes())
    out.append(h.hexdigest())
print(" ".join(out))
"""


def test_gate_bitwise_independent_of_cluster_size():
    digests = {}
    for c in ("1", "2", "4"):
        env = dict(os.environ, MOE_GATE_CLUSTER=c)
        r = subprocess.run([sys.executable, "-c", _SCRIPT % ROOT], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests[c] = r.stdout.split()
    assert digests["1"] == digests["2"] == digests["4"]
