"""Expert parallelism with the exchange over peer memory (moe_ep_*,
csrc/ep_p2p.cu): counts published into the peers' windows, token rows stored
straight into the owner's receive buffer, outputs read back from the owners'
windows by the combine.  No NCCL and no host sync on the data path.

The test box has one B200, so the 2-rank case runs two processes on the same
GPU: the windows are shared through CUDA IPC exactly as between two GPUs of an
NVSwitch box (only the link differs).  Parity: the sharded layer reproduces the
single-GPU layer bit for bit (routing and outputs), the receive layout equals
the host restatement (ep.recv_layout) and the exchange counts equal the
reference's plan_dynamic_exchange payload phase.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
SEED = 2303061820


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _single_gpu_reference(S, TD, HD, E, k):
    from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights

    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    x = make_tokens(S, TD, seed=SEED)
    layer = MoeLayer(shape, S, weights=w, keep_logits=False)
    ref = layer(x)
    torch.cuda.synchronize()
    v = layer.view()
    out = ref.view(torch.int16).cpu().numpy(), v["idx"].reshape(S, k).cpu().numpy()
    layer.close()
    return out


def _build(rank, world, S, TD, HD, E, k, placement, max_recv_rows=0, transport="p2p"):
    from paper_2303_06182_b200.ep import PeerExpertParallelMoE
    from paper_2303_06182_b200.layer import Context, LayerShape, make_tokens, make_weights

    ctx = Context.get(0)
    shape = LayerShape(TD, HD, E, k)
    Wg, W1, W2 = make_weights(shape, seed=SEED, ctx=ctx)
    x = make_tokens(S, TD, seed=SEED, ctx=ctx)
    loc = torch.from_numpy(placement.local_experts(rank)).long().cuda()
    mine = torch.arange(rank, S, world, device="cuda")  # token t lives on t % D (exchange.cpp:35-37)
    xl = x[mine].contiguous()
    ep = PeerExpertParallelMoE(ctx, placement, shape, Wg, W1[loc].contiguous(), W2[loc].contiguous(),
                               xl.shape[0], rank, max_recv_rows=max_recv_rows, transport=transport)
    return ep, x, xl, mine


@pytest.mark.parametrize("S,TD,HD,E,k,tile_n", [(1024, 256, 512, 16, 2, "128"),
                                                (1024, 256, 512, 16, 2, "256"),
                                                (4096, 1024, 4096, 8, 2, "")])
def test_peer_ep_one_rank_bitwise_equals_layer(S, TD, HD, E, k, tile_n, monkeypatch):
    """World size 1 (the exchange goes through the rank's own window); 128- and
    256-token work items (the receive FFN's N), auto = 256 at 1024 rows/expert."""
    from paper_2303_06182_b200.ep import Placement

    if tile_n:
        monkeypatch.setenv("MOE_EP_TILE_N", tile_n)
    ref_bits, ref_idx = _single_gpu_reference(S, TD, HD, E, k)
    ep, x, xl, mine = _build(0, 1, S, TD, HD, E, k, Placement.contiguous(E, 1))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        outs = [ep.forward(xl, s).clone() for _ in range(3)]
        out_g = torch.empty_like(xl)
        for _ in range(3):
            ep.forward(xl, s, out=out_g, graph=True)
    s.synchronize()
    ep.check_errors(s)
    for o in outs + [out_g]:
        assert (o.view(torch.int16).cpu().numpy() == ref_bits).all()
    v = ep.view(S)
    assert (v["idx"].cpu().numpy() == ref_idx).all()
    assert v["recv_rows"] == S * k
    ep.close()


def test_peer_ep_capacity_overflow_is_reported():
    from paper_2303_06182_b200._capi import MoeError
    from paper_2303_06182_b200.ep import Placement

    S, TD, HD, E, k = 512, 256, 512, 8, 2
    ep, x, xl, mine = _build(0, 1, S, TD, HD, E, k, Placement.contiguous(E, 1), max_recv_rows=100)
    ep.forward(xl)
    with pytest.raises(MoeError, match="receive capacity"):
        ep.check_errors()
    ep.close()


@pytest.mark.parametrize("S,TD,HD,E,k", [(1024, 256, 512, 16, 2), (333, 256, 512, 12, 3),
                                         (16384, 1024, 4096, 512, 2)])
def test_nccl_ep_one_rank_bitwise_equals_layer(S, TD, HD, E, k):
    """The C ABI's NCCL transport (csrc/ep_nccl.cu: count all-gather, host
    sync, grouped ncclSend/ncclRecv of the rows and weights, regroup by local
    expert, fused FFN, reverse send/recv, combine) at world size 1 -- the
    rank's sends go to itself through NCCL -- reproduces the single-GPU layer
    bit for bit, eagerly and through the graph entry point (which runs NCCL
    forwards eagerly)."""
    from paper_2303_06182_b200.ep import Placement

    ref_bits, ref_idx = _single_gpu_reference(S, TD, HD, E, k)
    ep, x, xl, mine = _build(0, 1, S, TD, HD, E, k, Placement.contiguous(E, 1), transport="nccl")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        outs = [ep.forward(xl, s).clone() for _ in range(2)]
        outs.append(ep.forward(xl, s, graph=True).clone())
        ep.enable_timing(True)
        outs.append(ep.forward(xl, s).clone())
        st = ep.stage_times()
    s.synchronize()
    ep.check_errors(s)
    for o in outs:
        assert (o.view(torch.int16).cpu().numpy() == ref_bits).all()
    v = ep.view(S)
    assert (v["idx"].cpu().numpy() == ref_idx).all()
    assert v["recv_rows"] == S * k
    assert all(t >= 0 for t in st.values()) and st["ffn"] > 0
    ep.close()


def test_nccl_ep_capacity_overflow_fails_the_forward():
    from paper_2303_06182_b200._capi import MoeError
    from paper_2303_06182_b200.ep import Placement

    S, TD, HD, E, k = 512, 256, 512, 8, 2
    ep, x, xl, mine = _build(0, 1, S, TD, HD, E, k, Placement.contiguous(E, 1), max_recv_rows=100,
                             transport="nccl")
    with pytest.raises(MoeError, match="receive capacity"):
        ep.forward(xl)
    ep.close()


def test_peer_ep_overflow_still_computes_the_rows_that_fit():
    """A receive capacity below the batch: the rows that fit are computed
    (the work list is clamped, not dropped), the overflow is reported, and a
    forward with enough capacity afterwards is exact."""
    from paper_2303_06182_b200._capi import MoeError
    from paper_2303_06182_b200.ep import Placement

    S, TD, HD, E, k = 512, 256, 512, 8, 2
    ref_bits, _ = _single_gpu_reference(S, TD, HD, E, k)
    ep, x, xl, mine = _build(0, 1, S, TD, HD, E, k, Placement.contiguous(E, 1), max_recv_rows=600)
    out = ep.forward(xl)
    with pytest.raises(MoeError, match="receive capacity"):
        ep.check_errors()
    v = ep.view(S)
    assert v["n_items"] > 0
    ok = v["dest"].cpu().numpy() >= 0  # sorted rows that were stored
    assert 0 < ok.sum() < S * k
    # tokens whose every row was stored are exact
    pos = np.empty(S * k, np.int64)
    pos[v["order"].cpu().numpy()] = np.arange(S * k)
    full = ok[pos.reshape(S, k)].all(axis=1)
    assert full.any()
    assert (out.view(torch.int16).cpu().numpy()[full] == ref_bits[full]).all()
    ep.close()


def _worker(rank, world, port, S, TD, HD, E, k, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), MOE_EP_TIMEOUT_MS="60000")
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_06182_b200.ep import Placement

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        loads = np.random.default_rng(5).random((E, 4))
        pl = Placement.greedy(loads, world)
        ep, x, xl, mine = _build(rank, world, S, TD, HD, E, k, pl)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        outs = []
        with torch.cuda.stream(s):
            for i in range(steps):
                outs.append(ep.forward(xl, s, graph=(i >= steps // 2)).clone())
        s.synchronize()
        ep.check_errors(s)
        v = ep.view(xl.shape[0])
        res = {
            "rank": rank, "mine": mine.cpu().numpy(), "device_of": pl.device_of,
            "outs": [o.view(torch.int16).cpu().numpy() for o in outs],
            "idx": v["idx"].cpu().numpy(), "counts": v["counts"].cpu().numpy(),
            "counts_all": v["counts_all"].cpu().numpy(), "dest": v["dest"].cpu().numpy(),
            "order": v["order"].cpu().numpy(), "recv_x": v["recv_x"].view(torch.int16).cpu().numpy(),
            "x_local": xl.view(torch.int16).cpu().numpy(),
        }
        q.put(res)
        ep.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,TD,HD,E,k,overlap", [(512, 256, 512, 16, 2, "0"), (4096, 1024, 4096, 64, 2, "0"),
                                                 (4096, 1024, 4096, 64, 2, "1")])
def test_peer_ep_two_ranks_bitwise_equals_single_gpu(S, TD, HD, E, k, overlap, monkeypatch):
    """overlap "1": expert-ordered dispatch with per-expert arrival counters
    and GEMM1 tiles waiting per expert (MOE_EP_OVERLAP)."""
    from paper_2303_06182_b200.ep import recv_layout
    from test_ep_gpu import collect

    monkeypatch.setenv("MOE_EP_OVERLAP", overlap)

    world, steps = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, TD, HD, E, k, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(collect(procs, q, world, 600), key=lambda r: r["rank"])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ref_bits, ref_idx = _single_gpu_reference(S, TD, HD, E, k)
    El = E // world
    # every rank holds the same count matrix; row s = rank s's counts
    ca = res[0]["counts_all"]
    for r in res:
        assert (r["counts_all"] == ca).all()
        assert (ca[r["rank"]] == r["counts"]).all()
    # routing and outputs: bitwise equal to the single-GPU layer, every step
    for r in res:
        assert (r["idx"] == ref_idx[r["mine"]]).all()
        for o in r["outs"]:
            assert (o == ref_bits[r["mine"]]).all()
    # exchange counts == the reference's plan (rows src -> dst)
    dev_of = res[0]["device_of"]
    key = np.empty(E, np.int64)
    for d in range(world):
        loc = np.nonzero(dev_of == d)[0]
        key[loc] = d * El + np.arange(len(loc))
    for r in res:
        want = np.bincount(key[r["idx"].reshape(-1)], minlength=E)
        assert (want == r["counts"]).all()
    # receive layout: row i of sender s with key q lands at start[s, e] + rank in segment
    starts = [recv_layout(ca, p, El) for p in range(world)]
    for r in res:
        src = r["rank"]
        splits = np.concatenate([[0], np.cumsum(r["counts"])])
        for i, (d, slot) in enumerate(zip(r["dest"], r["order"])):
            qk = np.searchsorted(splits, i, side="right") - 1
            p, e = divmod(qk, El)
            row = starts[p][src, e] + (i - splits[qk])
            assert d == (p << 28) | row
            assert (res[p]["recv_x"][row] == r["x_local"][slot // k]).all()


def _timeout_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), MOE_EP_TIMEOUT_MS="1500")
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_06182_b200._capi import MOE_ERR_PEER_TIMEOUT, MoeError
    from paper_2303_06182_b200.ep import Placement

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        S, TD, HD, E, k = 256, 256, 512, 8, 2
        ep, x, xl, mine = _build(rank, world, S, TD, HD, E, k, Placement.contiguous(E, world))
        status = 0
        if rank == 0:  # rank 1 never calls forward: rank 0's waits must time out, not hang
            ep.forward(xl)
            try:
                ep.check_errors()
            except MoeError as e:
                status = e.status
        dist.barrier()
        q.put((rank, status))
        ep.close()
    finally:
        dist.destroy_process_group()


def test_peer_ep_missing_peer_times_out_instead_of_hanging():
    from paper_2303_06182_b200._capi import MOE_ERR_PEER_TIMEOUT
    from test_ep_gpu import collect

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(collect(procs, q, 2, 300))
    for p in procs:
        p.join(120)
    assert res[0] == MOE_ERR_PEER_TIMEOUT


@pytest.mark.parametrize("world,transport", [(1, "p2p"), (2, "p2p"), (4, "p2p"), (1, "nccl")])
def test_cxx_host_expert_parallel_demo(world, transport, tmp_path):
    """Pure C++ host (include/moesim/gpu_layer.hpp ExpertParallelLayer), ranks
    forked by tools/ep_p2p_demo.cpp, handles (p2p) or the NCCL unique id
    exchanged through files; every rank's rows bitwise equal to the
    single-GPU layer.  NCCL refuses two ranks on one GPU: world 1 here."""
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "bin",
                       "ep_p2p_demo")
    r = subprocess.run([exe, "--world", str(world), "--tokens", "1024", "--experts", "32",
                        "--transport", transport, "--dir", str(tmp_path / "ep")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 rows differ" in r.stdout
