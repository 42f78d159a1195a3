"""Expert parallelism with the real kernels: 2 ranks sharing the one B200 of the
test box (the gpurun box has a single GPU; NCCL refuses two ranks on one
device, so the transport is gloo with host staging -- the exchange logic and
every kernel are the production ones).  The sharded layer must reproduce the
single-GPU layer: same routing bit-for-bit, same outputs (each row's FFN is
computed by the same tcgen05 kernel with the same K order, so the results are
expected to be bitwise equal).
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


def _worker(rank, world, port, S, TD, HD, E, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2303_06182_b200.ep import ExpertParallelMoE, KernelBackend, Placement, Transport
    from paper_2303_06182_b200.layer import Context, LayerShape, make_tokens, make_weights

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        ctx = Context.get(0)
        shape = LayerShape(TD, HD, E, k)
        Wg, W1, W2 = make_weights(shape, seed=SEED, ctx=ctx)
        x = make_tokens(S, TD, seed=SEED, ctx=ctx)
        loads = np.random.default_rng(5).random((E, 4))
        pl = Placement.greedy(loads, world)
        loc = torch.from_numpy(pl.local_experts(rank)).long().cuda()
        be = KernelBackend(ctx, shape, Wg, W1[loc].contiguous(), W2[loc].contiguous(), S, S * k)
        layer = ExpertParallelMoE(pl, k, be, Transport(), rank)
        mine = torch.arange(rank, S, world, device="cuda")
        out = layer.forward(x[mine].contiguous())
        torch.cuda.synchronize()
        be.check_errors(None)
        q.put((rank, mine.cpu().numpy(), out.view(torch.int16).cpu().numpy(),
               layer.last["idx"].cpu().numpy()))
        be.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("S,TD,HD,E,k", [(512, 256, 512, 16, 2), (4096, 1024, 4096, 64, 2)])
def test_expert_parallel_two_ranks_matches_single_gpu(S, TD, HD, E, k):
    from paper_2303_06182_b200.layer import LayerShape, MoeLayer, make_tokens, make_weights

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, S, TD, HD, E, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = collect(procs, q, world, 600)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    shape = LayerShape(TD, HD, E, k)
    w = make_weights(shape, seed=SEED)
    x = make_tokens(S, TD, seed=SEED)
    layer = MoeLayer(shape, S, weights=w, keep_logits=False)
    ref = layer(x)
    torch.cuda.synchronize()
    v = layer.view()
    ref_bits = ref.view(torch.int16).cpu().numpy()
    ref_idx = v["idx"].reshape(S, k).cpu().numpy()
    got = np.zeros_like(ref_bits)
    got_idx = np.zeros_like(ref_idx)
    for rank, mine, o, ix in res:
        got[mine] = o
        got_idx[mine] = ix
    assert (got_idx == ref_idx).all()
    diff = (got != ref_bits).sum()
    if diff:
        a = torch.from_numpy(got).view(torch.bfloat16).float()
        b = torch.from_numpy(ref_bits).view(torch.bfloat16).float()
        rel = float((a - b).norm() / b.norm())
        print(f"EP vs single-GPU: {diff} bf16 values differ, rel_fro={rel:.2e}")
        assert rel < 1e-3
