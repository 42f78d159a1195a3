"""CPU tests: pin the oracle before trusting it.

* the C restatement (oracle/routing_oracle.c) and the verbatim reference build
  (oracle/_ref) agree with the reference's golden vectors (tests/golden, made by
  tests/golden/make_golden.py from the reference itself) and with each other
  on the reference's randomized suites;
* the numpy layer oracle's conventions (ties, slot order, weights) hold;
* the counter-based synthetic generator is exact and well-distributed.
No GPU is touched here.
"""
import hashlib

import numpy as np
import pytest

from oracle import layer as OL
from oracle import native as N
from refrng import MT19937_64, experts_array, random_batch

needs_ref = pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")


def _digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
        h.update(b"|")
    return h.hexdigest()


# ------------------------------------------------------------ golden vectors
def test_c_oracle_explicit_goldens(golden):
    for c in golden["explicit"]:
        ex = np.array(c["experts"], np.int32)
        if c["kind"] == "dynamic":
            o, cnt, s, pos = N.c_dynamic_dispatch(ex, c["E"])
            assert o.tolist() == c["expect"]["order"], c["src"]
            assert cnt.tolist() == c["expect"]["counts"], c["src"]
            assert s.tolist() == c["expect"]["splits"], c["src"]
            assert (o[pos] == np.arange(ex.size)).all()
        elif c["kind"] == "static":
            cap, slots, dropped, pos = N.c_static_dispatch(ex, c["E"], c["C"])
            assert cap == c["expect"]["capacity"], c["src"]
            assert slots.tolist() == c["expect"]["slots"], c["src"]
            assert dropped.tolist() == c["expect"]["dropped"], c["src"]


def test_golden_values_match_reference_test_assertions(golden):
    """The fixture must hold what test_gating.cpp asserts (guards the generator)."""
    ex = {c["src"] + c["kind"]: c for c in golden["explicit"]}
    d = ex["test_gating.cpp:132-138dynamic"]["expect"]
    assert d["counts"] == [3, 1, 2] and d["splits"] == [0, 3, 4, 6] and d["order"] == [1, 3, 5, 2, 0, 4]
    s = ex["test_gating.cpp:64-77static"]["expect"]
    assert s["slots"] == [[1, 3, 5], [2, -1, -1], [0, 4, -1]]
    s = ex["test_gating.cpp:79-85static"]["expect"]
    assert s["slots"][0] == [0, 1, 2] and s["dropped"] == [[3, 0]]
    assert ex["test_gating.cpp:149-158dynamic"]["expect"]["order"] == [0, 3, 1, 2]
    assert ex["test_gating.cpp:292-302debug_json_dynamic"]["expect"] == (
        '{"counts":[1,2],"num_experts":2,"order":[1,0,2],"seq_len":3,"splits":[0,1,3],"top_k":1}')
    st = ex["test_gating.cpp:292-302debug_json_static"]["expect"]
    assert '"capacity":1' in st and '"dropped":[[2,1]]' in st
    caps = {(c, s): v for c, s, v in golden["scalars"]["expert_capacity"]}
    assert caps[(0.5, 6)] == 3 and caps[(0.05, 2048)] == 103 and caps[(0.1, 30)] == 3
    assert caps[(1.0, 128)] == 128 and caps[(0.3, 5)] == 2 and caps[(0.05, 16384)] == 820
    masks = {(s, e, c): v for s, e, c, v in golden["scalars"]["dispatch_mask_elements"]}
    assert masks[(6, 3, 0.5)] == 54 and masks[(2048, 512, 0.05)] == 108003328


def test_c_oracle_scalars(golden):
    lib = N.c_oracle()
    for c, s, v in golden["scalars"]["expert_capacity"]:
        assert lib.or_expert_capacity(c, s) == v
    for e, c, k, v in golden["scalars"]["waste_factor"]:
        assert abs(lib.or_waste_factor(e, c, k) - v) <= 1e-12 * abs(v)
    for s, e, c, v in golden["scalars"]["dispatch_mask_elements"]:
        assert lib.or_dispatch_mask_elements(s, e, c) == v


def _replay(name, seed, iters, fn):
    rng = MT19937_64(seed)
    arrays = []
    for _ in range(iters):
        item = fn(rng)
        if item is None:
            continue
        kind, ex, E, C = item
        if kind == "dynamic":
            o, c, s, _ = N.c_dynamic_dispatch(ex, E)
            arrays += [o, c, s]
        else:
            cap, slots, dropped, _ = N.c_static_dispatch(ex, E, C)
            arrays += [np.array([cap]), slots.reshape(-1), dropped.reshape(-1)]
    return _digest(arrays)


def test_c_oracle_random_suites_match_reference_digests(golden):
    gens = {}

    def g_drop(rng):
        E, k, S = 2 + rng() % 8, 1 + rng() % 2, 1 + rng() % 40
        C = 0.05 + (rng() % 100) / 100.0
        return ("static", experts_array(random_batch(rng, S, E, k)), E, C)

    def g_dyn(rng):
        E, k, S = 2 + rng() % 16, 1 + rng() % 2, 1 + rng() % 60
        return ("dynamic", experts_array(random_batch(rng, S, E, k)), E, 0.0)

    def g_acc(rng):
        E, k, S = 2 + rng() % 31, 1 + rng() % 2, 1 + rng() % 256
        return ("dynamic", experts_array(random_batch(rng, S, E, k)), E, 0.0)

    gens = {"drop_law": g_drop, "dynamic_scan": g_dyn, "acceptance_routing": g_acc}
    for suite in golden["random"]:
        got = _replay(suite["name"], suite["seed"], suite["iters"], gens[suite["name"]])
        assert got == suite["digest"], suite["name"]


@needs_ref
def test_c_oracle_matches_reference_large():
    rng = np.random.default_rng(5)
    for S, E, k in [(2048, 8, 1), (16384, 512, 2), (6144, 128, 2), (1, 4, 1), (777, 13, 3)]:
        ex = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
        ro, rc, rs = N.ref_dynamic_dispatch(ex, E)
        co, cc, cs, _ = N.c_dynamic_dispatch(ex, E)
        assert (ro == co).all() and (rc == cc).all() and (rs == cs).all()
        for C in (0.05, 0.5, 1.0):
            rcap, rsl, rdr = N.ref_static_dispatch(ex, E, C)
            ccap, csl, cdr, _ = N.c_static_dispatch(ex, E, C)
            assert rcap == ccap and (rsl == csl).all() and (rdr == cdr).all()


@needs_ref
def test_reference_error_messages():
    ex = np.zeros((2, 1), np.int32)
    with pytest.raises(N.OracleError, match="num_experts must be positive"):
        N.ref_dynamic_dispatch(ex, 0)
    with pytest.raises(N.OracleError, match="top_k exceeds num_experts"):
        N.ref_dynamic_dispatch(np.zeros((2, 3), np.int32), 2)
    with pytest.raises(N.OracleError, match="dynamic_dispatch requires dynamic mode"):
        N.ref_dynamic_dispatch(ex, 2, mode_static=True)
    with pytest.raises(N.OracleError, match="static_dispatch requires static mode"):
        N.ref_static_dispatch(ex, 2, 1.0, mode_static=False)
    with pytest.raises(N.OracleError, match="capacity factor must be positive in static mode"):
        N.ref_static_dispatch(ex, 2, 0.0)


@needs_ref
def test_reference_combine_is_inverse_permutation():
    """gating.hpp:107-141: the C oracle's pos[] reproduces the reference combine."""
    rng = MT19937_64(11)
    b = random_batch(rng, 32, 8, 2)
    ex = experts_array(b)
    order, _, _ = N.ref_dynamic_dispatch(ex, 8)
    w = np.array([ta.weights for ta in b.tokens])
    n, oe, ow, op = N.ref_combine_dynamic(ex, w, 8, order)
    _, _, _, pos = N.c_dynamic_dispatch(ex, 8)
    assert (n == 2).all()
    assert (op.reshape(-1) == order[pos]).all()
    assert (oe == ex).all() and (ow == w).all()


@needs_ref
def test_exchange_counts_oracle_matches_reference():
    rng = np.random.default_rng(3)
    for D in (2, 4, 8):
        E, S, k = 64, 1000, 2
        ex = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
        dev = N.ref_greedy_place(rng.random((E, 6)), D)
        size_b, pay_b = N.ref_plan_dynamic_exchange(ex, E, D, dev, 2048)
        cnt = N.c_exchange_counts(ex, D, dev)
        assert (pay_b == cnt * 2048).all()
        assert size_b.sum() == D * E * 4  # test_exchange.cpp:133-135


# ------------------------------------------------------------ layer oracle
def test_topk_ties_lower_id_and_slot_order():
    L = np.array([[1.0, 3.0, 3.0, 2.0], [0.5, 0.5, 0.5, 0.5], [4.0, 1.0, 5.0, 5.0]], np.float32)
    idx, w = OL.topk_from_logits(L, 2)
    assert idx.tolist() == [[1, 2], [0, 1], [2, 3]]
    assert np.allclose(w.sum(1), 1.0, atol=0, rtol=0) or np.abs(w.sum(1) - 1).max() < 1e-15
    assert np.allclose(w[1], [0.5, 0.5])
    idx1, w1 = OL.topk_from_logits(L, 1)
    assert idx1[:, 0].tolist() == [1, 0, 2] and (w1 == 1.0).all()


def test_topk_weights_are_restricted_softmax():
    rng = np.random.default_rng(0)
    L = rng.standard_normal((50, 16)).astype(np.float32)
    idx, w = OL.topk_from_logits(L, 3)
    for t in range(50):
        p = np.exp(L[t].astype(np.float64) - L[t].max())
        p /= p.sum()
        sel = p[idx[t]]
        assert np.allclose(w[t], sel / sel.sum(), rtol=1e-12, atol=1e-14)
        assert (np.diff(L[t, idx[t]]) <= 0).all()


def test_synth_is_exact_and_uniform():
    x = OL.synth_f32(200000, 7, OL.T_X, 1.5)
    assert x.dtype == np.float32
    assert x.min() >= -1.5 and x.max() < 1.5
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1.5 ** 2 / 3) < 0.01
    # counter-based: a slice equals the same indices generated directly
    idx = np.arange(1000, 1100, dtype=np.uint64)
    assert (OL.synth_f32(idx, 7, OL.T_X, 1.5) == x[1000:1100]).all()
    # different tensor ids decorrelate
    y = OL.synth_f32(200000, 7, OL.T_W1, 1.5)
    assert abs(np.corrcoef(x, y)[0, 1]) < 0.01


def test_bf16_round_nearest_even():
    vals = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e38, 1e-40], np.float32)
    b = OL.bf16_round(vals)
    back = OL.bf16_to_f32(b)
    assert back[0] == 1.0
    assert back[1] == 1.0          # halfway 1 + 2^-8 -> even (1.0)
    assert back[2] == 1.015625     # halfway 1 + 3*2^-8 -> even (1 + 2^-6)
    assert back[3] == -2.5


def test_layer_oracle_k1_identity_expert():
    """With W2 = W1^T and W1 = I-like, y = relu(x): checks plumbing and combine."""
    TD = HD = 8
    E = 2
    X = np.linspace(-1, 1, 3 * TD, dtype=np.float32).reshape(3, TD)
    W1 = np.stack([np.eye(HD, TD, dtype=np.float32)] * E)
    W2 = np.stack([np.eye(TD, HD, dtype=np.float32)] * E)
    idx = np.array([[0], [1], [0]], np.int32)
    w = np.ones((3, 1))
    out = OL.layer_forward(X, W1, W2, idx, w, E)
    assert np.allclose(out, np.maximum(X, 0))


@needs_ref
@pytest.mark.parametrize("S,TD,HD,E,k", [(64, 32, 48, 8, 2), (50, 16, 16, 6, 3), (40, 24, 32, 5, 1)])
def test_layer_oracle_combine_equals_reference_dispatch_and_combine(S, TD, HD, E, k):
    """Pins the oracle's dispatch -> FFN -> weighted-combine plumbing to the
    reference where the reference has semantics: expert rows are computed in
    the reference's dynamic_dispatch order (gating.cpp:58-86) and each
    token's output is summed over the entries the reference's combine<T>
    returns (gating.hpp:107-141: slot order, the routing weights), payload =
    the row index of that slot's expert output.  Same fp32 operations ->
    bitwise equal to oracle.layer.layer_forward."""
    rng = np.random.default_rng(S * 1000 + E)
    X = rng.standard_normal((S, TD)).astype(np.float32)
    W1 = (rng.standard_normal((E, HD, TD)) / np.sqrt(TD)).astype(np.float32)
    W2 = (rng.standard_normal((E, TD, HD)) / np.sqrt(HD)).astype(np.float32)
    idx, w = OL.topk_from_logits(rng.standard_normal((S, E)).astype(np.float32), k)
    order, counts, splits = N.ref_dynamic_dispatch(idx, E, w)
    # expert FFN over the reference's expert-grouped rows
    Y = np.zeros((S * k, TD), np.float32)
    for e in range(E):
        rows = order[splits[e]:splits[e + 1]]
        if len(rows):
            Y[splits[e]:splits[e + 1]] = OL.expert_ffn(X[rows // k], W1[e], W2[e])
    n, oe, ow, op = N.ref_combine_dynamic(idx, w, E, np.arange(S * k, dtype=np.int32))
    assert (n == k).all() and (oe == idx).all()
    out = np.zeros((S, TD), np.float32)
    for j in range(k):  # the reference's presentation order == slot order
        out += ow[:, j].astype(np.float32)[:, None] * Y[op[:, j]]
    ref = OL.layer_forward(X, W1, W2, idx, w, E)
    assert np.array_equal(out, ref)


@needs_ref
def test_reference_routing_timer_runs_the_reference_functions():
    """oracle/ref_capi.cpp ref_time_routing (bench.py cpu_baseline's routing
    numbers): every timed function ran (positive times), the static ones only
    when a capacity factor is given."""
    rng = np.random.default_rng(5)
    S, k, E = 4096, 2, 64
    ex = np.stack([rng.permutation(E)[:k] for _ in range(S)]).astype(np.int32)
    w = np.full((S, k), 0.5)
    t = N.ref_time_routing(ex, w, E, 0.0, reps=2)
    assert set(t) == {"dynamic_dispatch", "combine_dynamic"} and all(v > 0 for v in t.values())
    t = N.ref_time_routing(ex, w, E, 0.25, reps=2)
    assert set(t) == {"dynamic_dispatch", "combine_dynamic", "static_dispatch", "combine_static"}
    assert all(v > 0 for v in t.values())
