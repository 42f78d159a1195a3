"""Expert parallelism over 2 processes (gloo, CPU): the production exchange
logic of paper_2303_06182_b200/ep.py (keyed dispatch -> count all-to-all ->
payload all-to-all -> remote experts -> reverse all-to-all -> combine) with
the CPU oracle as the compute backend (tests only).

Checks, on a global batch spread round robin over D ranks (exchange.cpp:35-37):
  * layer output == the single-process oracle layer (same routing)
  * per-(src, dst) slot counts == the reference's plan_dynamic_exchange payload
    bytes / token_bytes (exchange.cpp:95-120), size phase == D*E*4 bytes
  * placement policies restate balance.cpp (greedy vs the verbatim build)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layer as OL
from oracle import native as N
from paper_2303_06182_b200.ep import ExpertParallelMoE, Placement, Transport

SEED = 7


def collect(procs, q, n, timeout):
    """Results of n worker processes; fails fast if a worker dies."""
    import queue
    import time

    out, t0 = [], time.time()
    while len(out) < n:
        try:
            out.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p for p in procs if p.exitcode not in (None, 0)]
            if dead:
                raise AssertionError(f"worker exited with code {dead[0].exitcode}")
            if time.time() - t0 > timeout:
                raise AssertionError("workers timed out")
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _weights(E, TD, HD):
    sc = OL.init_scales(TD, HD)
    Wg = OL.bf16_to_f32(OL.synth_bf16((E, TD), SEED, OL.T_WG, sc["wg"]))
    W1 = OL.bf16_to_f32(OL.synth_bf16((E, HD, TD), SEED, OL.T_W1, sc["w1"]))
    W2 = OL.bf16_to_f32(OL.synth_bf16((E, TD, HD), SEED, OL.T_W2, sc["w2"]))
    X = OL.bf16_to_f32(OL.synth_bf16((64, TD), SEED, OL.T_X, sc["x"]))
    return Wg, W1, W2, X


class OracleBackend:
    """CPU stand-in for KernelBackend, built from the oracle (tests only)."""

    def __init__(self, Wg, W1_local, W2_local):
        self.Wg, self.W1, self.W2 = Wg, W1_local, W2_local

    def gate(self, x, k, stream):
        logits = OL.gate_logits(x.numpy(), self.Wg)
        idx, w = OL.topk_from_logits(logits, k)
        return torch.from_numpy(idx), torch.from_numpy(w.astype(np.float32))

    def route_keyed(self, idx, w, key_map, n_keys, stream):
        keys = key_map.numpy()[idx.numpy()]
        order, counts, splits, pos = N.c_dynamic_dispatch(keys, n_keys)
        wpos = w.numpy().reshape(-1)[order]
        return (torch.from_numpy(counts.copy()), torch.from_numpy(order.copy()),
                torch.from_numpy(pos.copy()), torch.from_numpy(wpos.astype(np.float32)))

    def gather(self, x, order, k, stream):
        return x[torch.from_numpy(order.numpy() // k).long()]

    def segment_keys(self, recv_counts_flat, mod, total, stream):
        c = recv_counts_flat.numpy()
        return torch.from_numpy(np.repeat(np.arange(c.size) % mod, c).astype(np.int32))

    def ffn(self, xr, keys, wr, stream):
        y = np.zeros(xr.shape, np.float32)
        xn, kn, wn = xr.numpy(), keys.numpy(), wr.numpy()
        for e in np.unique(kn):
            m = kn == e
            y[m] = OL.expert_ffn(xn[m], self.W1[e], self.W2[e]) * wn[m][:, None]
        return torch.from_numpy(y)

    def combine(self, yb, pos, S, k, stream):
        p = pos.numpy().reshape(S, k)
        y = yb.numpy()
        out = np.zeros((S, yb.shape[1]), np.float32)
        for j in range(k):
            out += y[p[:, j]]
        return torch.from_numpy(out)


def _worker(rank, world, port, E, k, TD, HD, placement_kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Wg, W1, W2, X = _weights(E, TD, HD)
        if placement_kind == "greedy":
            loads = np.random.default_rng(3).random((E, 5))
            pl = Placement.greedy(loads, world)
        else:
            pl = Placement.contiguous(E, world)
        loc = pl.local_experts(rank)
        be = OracleBackend(Wg, W1[loc], W2[loc])
        layer = ExpertParallelMoE(pl, k, be, Transport(), rank, device="cpu")
        mine = np.arange(rank, X.shape[0], world)  # token t lives on rank t % D
        out = layer.forward(torch.from_numpy(X[mine]))
        q.put((rank, mine, out.numpy(), layer.last["send_counts"].numpy(),
               layer.last["idx"].numpy(), pl.device_of))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("placement_kind", ["contiguous", "greedy"])
def test_expert_parallel_matches_single_process(placement_kind):
    world, E, k, TD, HD = 2, 8, 2, 32, 48
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, k, TD, HD, placement_kind, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = collect(procs, q, world, 120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    Wg, W1, W2, X = _weights(E, TD, HD)
    S = X.shape[0]
    out = np.zeros((S, TD), np.float32)
    idx = np.zeros((S, k), np.int32)
    counts = {}
    device_of = None
    for rank, mine, o, sc, ix, dev in res:
        out[mine] = o
        idx[mine] = ix
        counts[rank] = sc.sum(1)  # slots rank -> each destination device
        device_of = dev
    # 1. layer output == single-process oracle with the same routing
    ridx, rw = OL.topk_from_logits(OL.gate_logits(X, Wg), k)
    assert (ridx == idx).all()
    ref = OL.layer_forward(X, W1, W2, ridx, rw, E)
    assert OL.rel_fro(out, ref) < 1e-5
    # 2. exchange counts == the reference's dynamic exchange plan
    mat = np.stack([counts[r] for r in range(world)])
    assert (mat == N.c_exchange_counts(idx, world, device_of)).all()
    if N.ref_available():
        size_b, pay_b = N.ref_plan_dynamic_exchange(idx, E, world, device_of, TD * 2)
        assert (pay_b == mat * TD * 2).all()
        assert size_b.sum() == world * E * 4


@pytest.mark.skipif(not N.ref_available(), reason="oracle/_ref not built")
def test_greedy_placement_restates_reference():
    rng = np.random.default_rng(11)
    for E, D in [(8, 2), (16, 4), (512, 8), (64, 8)]:
        loads = rng.random((E, 7))
        loads[rng.integers(0, E, 3)] = loads[0]  # ties in mean load
        assert (Placement.greedy(loads, D).device_of == N.ref_greedy_place(loads, D)).all()
    assert (Placement.contiguous(16, 4).device_of == N.ref_contiguous_place(16, 4)).all()
    # test_balance.cpp:102-122 goldens
    h = np.array([[0.4], [0.3], [0.2], [0.1]])
    assert Placement.greedy(h, 2).device_of.tolist() == [0, 1, 1, 0]
    u = np.full((4, 1), 0.25)
    assert Placement.greedy(u, 2).device_of.tolist() == [0, 1, 0, 1]


def test_placement_key_map_groups_devices():
    pl = Placement(np.array([1, 0, 1, 0, 0, 1], np.int32), 2)
    km = pl.key_map()
    # device 0 holds experts 1,3,4 -> keys 0,1,2 ; device 1 holds 0,2,5 -> keys 3,4,5
    assert km.tolist() == [3, 0, 4, 1, 2, 5]
    with pytest.raises(ValueError):
        Placement(np.array([0, 0, 0, 1], np.int32), 2).validate()


def test_peer_recv_layout_partitions_rows():
    """ep.recv_layout (the host restatement of ep_dispatch_kernel's destination
    rows): at every device the (source, local expert) segments tile [0, R)
    without gaps, ordered by local expert, then source rank -- the order the
    single-GPU layer gives the same rows (stable sort by expert of slots, and
    global slot order interleaves sources only within an expert)."""
    from paper_2303_06182_b200.ep import recv_layout

    rng = np.random.default_rng(3)
    for D, El in [(1, 4), (2, 8), (4, 16), (8, 64)]:
        ca = rng.integers(0, 50, size=(D, D * El))
        ca[:, rng.integers(0, D * El, 3)] = 0  # empty segments
        for p in range(D):
            st = recv_layout(ca, p, El)
            c = ca[:, p * El:(p + 1) * El]
            seg = sorted((int(st[s, e]), int(c[s, e]), e, s) for s in range(D) for e in range(El))
            pos = 0
            for start, n, e, s in seg:
                assert start == pos
                pos += n
            assert pos == c.sum()
            order = [(e, s) for _, n, e, s in sorted((int(st[s, e]), int(c[s, e]), e, s)
                                                      for s in range(D) for e in range(El)) if n]
            assert order == sorted(order)
