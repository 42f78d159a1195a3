"""The drop-in's adjacent API (exchange / balance / buffer) against the reference.

1. The reference's own unit tests -- proj/tests/test_{exchange,balance,buffer}.cpp
   -- compiled UNMODIFIED against include/moesim/*.hpp and libmoesim_b200
   (__graft_entry__._build_reference_tests).  test_balance / test_buffer are
   host policy and run here; test_exchange's dynamic plans come from the GPU
   (moe_exchange_counts_host), so it runs on the B200.
2. Randomised bit-exact checks of the C entry points against the verbatim
   reference build (oracle/_ref): placement (greedy / anticorr / Pearson /
   eval_balance) and the cache controller (moe_cache_policy_access, the code
   the GPU expert cache runs) for LIFO, FIFO and MIN.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import native as N
from paper_2303_06182_b200 import _capi, placement

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_tests")
need_ref = pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")


def _run_suite(name):
    exe = os.path.join(BIN, f"{name}_b200")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-1500:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed" in r.stdout


@pytest.mark.parametrize("name", ["test_balance", "test_buffer"])
def test_reference_suite_unmodified_host(name):
    _run_suite(name)


@pytest.mark.gpu
def test_reference_suite_unmodified_exchange_gpu():
    _run_suite("test_exchange")


def _random_history(rng, E, B, zero_rows=0):
    h = rng.random((E, B))
    if zero_rows:
        h[rng.choice(E, zero_rows, replace=False)] = 0.0
    h[rng.integers(0, E, 2)] = h[0]  # equal means and perfectly correlated rows
    return h / h.sum(axis=0, keepdims=True)


@need_ref
def test_placement_policies_bit_exact_vs_reference():
    rng = np.random.default_rng(2023)
    for E, D, B in [(8, 2, 3), (16, 4, 7), (64, 8, 16), (128, 8, 32), (512, 8, 8), (6, 3, 2)]:
        h = _random_history(rng, E, B, zero_rows=E // 8)
        g = placement.greedy_place(h, D)
        assert (g == N.ref_greedy_place(h, D)).all()
        for w in (0.0, 0.5, 2.0):
            assert (placement.anticorr_place(h, D, w) == N.ref_anticorr_place(h, D, w)).all()
        assert (placement.pearson_corr(h) == N.ref_pearson_corr(h)).all()
        for dev in (g, placement.contiguous_place(E, D)):
            rep = placement.eval_balance(dev, D, h)
            assert (rep["max_load"], rep["avg_max_load"], rep["objective"]) == N.ref_eval_balance(dev, D, h)
            assert np.allclose(rep["device_load"].sum(axis=0), 1.0)
    with pytest.raises(placement.PlacementError, match="divisible"):
        placement.greedy_place(np.ones((10, 2)), 4)
    with pytest.raises(placement.PlacementError, match="at least 2 batches"):
        placement.pearson_corr(np.ones((4, 1)))


@need_ref
def test_two_half_protocol_on_skewed_trace():
    """The reference CLI's balance study (tools/moesim.cpp:451-492): place on
    the first half of a skewed trace, score on the second.  Greedy and anticorr
    beat contiguous, and every number equals the reference's."""
    E, k, B, S = 128, 2, 40, 512
    ex, _ = N.ref_gen_synthetic_trace(E, k, B, S, 1.2, 0.9, 1.0, 31)
    loads = np.zeros((E, B))
    for b in range(B):
        loads[:, b] = np.bincount(ex.reshape(B, S * k)[b], minlength=E) / (S * k)
    train, test = loads[:, : B // 2], loads[:, B // 2:]
    D = 8
    res = {}
    for name, dev in (("contiguous", placement.contiguous_place(E, D)),
                      ("greedy", placement.greedy_place(train, D)),
                      ("anticorr", placement.anticorr_place(train, D))):
        rep = placement.eval_balance(dev, D, test)
        assert (rep["max_load"], rep["avg_max_load"], rep["objective"]) == N.ref_eval_balance(dev, D, test)
        res[name] = rep["avg_max_load"]
    print(res)
    assert res["greedy"] < res["contiguous"] and res["anticorr"] < res["contiguous"]


def _policy_access(resident, cache_size, policy, active, future):
    lib = _capi.load()
    res = np.zeros(cache_size + 1, np.int32)
    res[: len(resident)] = resident
    n = C.c_int(len(resident))
    a = np.ascontiguousarray(active, np.int32)
    f = None if future is None else np.ascontiguousarray(future, np.int32)
    st = np.zeros(4, np.int32)
    _capi.check(lib.moe_cache_policy_access(res.ctypes.data_as(C.c_void_p), C.byref(n), cache_size, policy,
                                            a.ctypes.data_as(C.c_void_p), a.size,
                                            None if f is None else f.ctypes.data_as(C.c_void_p),
                                            -1 if f is None else f.size, st.ctypes.data_as(C.c_void_p)))
    return tuple(int(x) for x in st), res[: n.value].tolist()


@need_ref
@pytest.mark.parametrize("policy", [0, 1, 2])
def test_cache_controller_bit_exact_vs_reference(policy):
    """moe_cache_policy_access (the GPU cache's controller) == access_batch of
    the verbatim reference build, batch by batch, on random access streams."""
    rng = np.random.default_rng(policy + 7)
    for _ in range(60):
        E = int(rng.integers(2, 40))
        cache = int(rng.integers(1, E + 1))
        batches = [np.sort(rng.choice(E, int(rng.integers(0, E + 1)), replace=False)) for _ in range(12)]
        flat = np.concatenate(batches) if batches else np.zeros(0, np.int32)
        starts = np.cumsum([0] + [len(b) for b in batches])
        ref = N.RefCache()
        mine = []
        for b, act in enumerate(batches):
            fut = flat[starts[b + 1]:] if policy == 2 else None
            rs, rres = ref.access(act, cache, policy, fut)
            ms, mine = _policy_access(mine, cache, policy, act, fut)
            assert ms == rs and mine == rres, (b, act.tolist())


def test_cache_controller_rejects_min_without_future():
    with pytest.raises(_capi.MoeInvalidArgument, match="future"):
        _policy_access([], 2, 2, [0, 1], None)
