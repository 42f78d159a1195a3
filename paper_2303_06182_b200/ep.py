"""Expert parallelism: the MoE layer sharded over D GPUs (one process each).

Mirrors the reference's simulated exchange (proj/src/exchange.cpp:95-120,
plan_dynamic_exchange) with real transfers:

  1. local gate + top-k, then dispatch keyed by (device, local expert) so the
     slots for every destination device are contiguous   (moe_route_dynamic_keyed)
  2. "size" phase: E/D int32 counts per (source, destination) pair
     (exchange.cpp:100-104) -- one all-to-all, then the single host sync of the
     layer (NCCL needs the split sizes on the host; PAPER.md:313's two-step design)
  3. "payload" phase: the token rows (bf16 TD) plus their gate weights go to
     the device that owns the expert (exchange.cpp:106-114), variable all-to-all
  4. the receiving device runs its local experts over the received rows
     (moe_ffn_forward: regroup by local expert, tcgen05 grouped FFN)
  5. the reverse all-to-all returns the expert outputs ("mirrors the forward
     plan transposed") and the origin combines them
     (moe_combine, slot order j)

Expert placement (`Placement`) is the reference's host-side policy
(balance.hpp:12-58): contiguous, or greedy by historical load.  Token residency
is round robin: global token t lives on device t % D (exchange.cpp:35-37).

The transport is torch.distributed (NCCL over NVLink on a B200 box; `gloo`
with host staging for CPU tests); the compute steps live in a backend object so
the exchange logic can be exercised on CPU with the oracle (tests only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _capi, placement
from ._capi import check


# ------------------------------------------------------------------ placement
@dataclass
class Placement:
    """Expert -> device with exactly E/D experts per device (balance.hpp:12-21)."""

    device_of: np.ndarray  # int32 [E]
    num_devices: int

    @property
    def num_experts(self) -> int:
        return int(self.device_of.size)

    @property
    def experts_per_device(self) -> int:
        return self.num_experts // self.num_devices

    def validate(self):
        """balance.cpp:42-57: every device holds exactly E/D experts."""
        E, D = self.num_experts, self.num_devices
        if D < 1 or E % D:
            raise ValueError("num_experts must divide evenly across devices")
        cnt = np.bincount(self.device_of, minlength=D)
        if (self.device_of < 0).any() or (self.device_of >= D).any() or (cnt != E // D).any():
            raise ValueError("placement must put exactly E/D experts on every device")

    def local_experts(self, d: int) -> np.ndarray:
        """Experts on device d, increasing id (their local index order)."""
        return np.nonzero(self.device_of == d)[0].astype(np.int32)

    def key_map(self) -> np.ndarray:
        """expert -> device * E/D + local index: the dispatch sort key."""
        El = self.experts_per_device
        key = np.empty(self.num_experts, np.int32)
        for d in range(self.num_devices):
            loc = self.local_experts(d)
            key[loc] = d * El + np.arange(len(loc), dtype=np.int32)
        return key

    # The policies are the C++ host library's (host/balance.cpp, the drop-in
    # of balance.cpp:59-151), bound through include/moesim/placement_c.h.
    @staticmethod
    def contiguous(E: int, D: int) -> "Placement":
        """balance.cpp:59-67: expert m on device floor(m / (E/D))."""
        p = Placement(placement.contiguous_place(E, D), D)
        p.validate()
        return p

    @staticmethod
    def greedy(loads: np.ndarray, D: int) -> "Placement":
        """balance.cpp:92-115: experts by mean historical load descending (ties:
        lower id) go to the open device with the least accumulated load (ties:
        lower device id); a device closes at E/D experts."""
        p = Placement(placement.greedy_place(loads, D), D)
        p.validate()
        return p

    @staticmethod
    def anticorr(loads: np.ndarray, D: int, weight: float = 0.5) -> "Placement":
        """balance.cpp:117-151: the greedy loop scored by sum over the
        device's experts of mean load + weight * Pearson correlation."""
        p = Placement(placement.anticorr_place(loads, D, weight), D)
        p.validate()
        return p

    def balance(self, loads: np.ndarray) -> dict:
        """eval_balance (balance.cpp:153-165) of this placement on a load history."""
        return placement.eval_balance(self.device_of, self.num_devices, loads)


# ------------------------------------------------------------------ transport
class Transport:
    """Variable all-to-all over torch.distributed.  With NCCL the tensors stay
    on the GPU (NVLink); with gloo they are staged through host memory."""

    def __init__(self, group=None):
        self.group = group
        self.backend = dist.get_backend(group)

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        if self.backend == "nccl":
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
            return out
        o = torch.empty(out.shape, dtype=out.dtype)
        i = inp.detach().cpu()
        dist.all_to_all_single(o, i, out_splits, in_splits, group=self.group)
        out.copy_(o)
        return out


# ------------------------------------------------------------------ compute backend
class KernelBackend:
    """The product: every step is a C-ABI call into libmoe_b200.so."""

    def __init__(self, ctx, shape, Wg, W1_local, W2_local, max_tokens, max_recv_rows, tile_n=0):
        self.ctx = ctx
        self.lib = ctx.lib
        self.shape = shape
        self.Wg = Wg
        # the FFN's TMA descriptors hold raw pointers: keep the tensors alive
        self.W1_local, self.W2_local = W1_local, W2_local
        E_l = W1_local.shape[0]
        d = _capi.FfnDesc(max_recv_rows, shape.token_dim, shape.hidden_dim, E_l, tile_n)
        h = C.c_void_p()
        check(self.lib.moe_ffn_create(ctx.h, C.byref(d), _p(W1_local), _p(W2_local), C.byref(h)))
        self.ffn_h = h
        self.max_recv_rows = max_recv_rows

    def close(self):
        if getattr(self, "ffn_h", None):
            self.lib.moe_ffn_destroy(self.ffn_h)
            self.ffn_h = None

    def gate(self, x, k, stream):
        S = x.shape[0]
        E = self.shape.num_experts
        idx = torch.empty(S, k, dtype=torch.int32, device=x.device)
        w = torch.empty(S, k, dtype=torch.float32, device=x.device)
        check(self.lib.moe_gate_topk(self.ctx.h, _p(x), _p(self.Wg), S, self.shape.token_dim, E, k,
                                     _p(idx), _p(w), None, _s(stream)))
        return idx, w

    def route_keyed(self, idx, w, key_map, n_keys, stream):
        S, k = idx.shape
        E = self.shape.num_experts
        dev = idx.device
        counts = torch.empty(n_keys, dtype=torch.int32, device=dev)
        splits = torch.empty(n_keys + 1, dtype=torch.int32, device=dev)
        order = torch.empty(S * k, dtype=torch.int32, device=dev)
        pos = torch.empty(S * k, dtype=torch.int32, device=dev)
        wpos = torch.empty(S * k, dtype=torch.float32, device=dev)
        check(self.lib.moe_route_dynamic_keyed(self.ctx.h, _p(idx), S, k, E, _p(key_map), n_keys,
                                               _p(counts), _p(splits), _p(order), _p(pos), _p(w),
                                               _p(wpos), _s(stream)))
        return counts, order, pos, wpos

    def gather(self, x, order, k, stream):
        rows = order.numel()
        xp = torch.empty(rows, x.shape[1], dtype=x.dtype, device=x.device)
        check(self.lib.moe_gather_rows(self.ctx.h, _p(x), _p(order), rows, k, x.shape[1], _p(xp),
                                       _s(stream)))
        return xp

    def segment_keys(self, recv_counts_flat, mod, total, stream):
        keys = torch.empty(max(total, 1), dtype=torch.int32, device=recv_counts_flat.device)
        check(self.lib.moe_fill_segments(self.ctx.h, _p(recv_counts_flat), recv_counts_flat.numel(),
                                         mod, _p(keys), _s(stream)))
        return keys[:total]

    def ffn(self, xr, keys, wr, stream):
        R = xr.shape[0]
        yr = torch.empty_like(xr)
        if R:
            if R > self.max_recv_rows:
                raise RuntimeError(f"received {R} rows > max_recv_rows {self.max_recv_rows}")
            check(self.lib.moe_ffn_forward(self.ffn_h, _p(xr), _p(keys), _p(wr), R, _p(yr), _s(stream)))
        return yr

    def combine(self, yb, pos, S, k, stream):
        out = torch.empty(S, yb.shape[1], dtype=yb.dtype, device=yb.device)
        check(self.lib.moe_combine(self.ctx.h, _p(yb), _p(pos), S, k, yb.shape[1], _p(out), _s(stream)))
        return out

    def check_errors(self, stream):
        check(self.lib.moe_check_errors(self.ctx.h, _s(stream)))


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _s(stream):
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------ the layer
class ExpertParallelMoE:
    """One rank's share of an expert-parallel MoE layer."""

    def __init__(self, placement: Placement, top_k: int, backend, transport: Transport, rank: int,
                 device="cuda"):
        placement.validate()
        self.placement = placement
        self.k = top_k
        self.backend = backend
        self.transport = transport
        self.rank = rank
        self.D = placement.num_devices
        self.E = placement.num_experts
        self.El = placement.experts_per_device
        self.device = torch.device(device)
        self.key_map = torch.from_numpy(placement.key_map()).to(self.device)
        self.last = {}

    def forward(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        B, k, D, El = self.backend, self.k, self.D, self.El
        S = x.shape[0]
        TD = x.shape[1]
        idx, w = B.gate(x, k, stream)
        counts, order, pos, wpos = B.route_keyed(idx, w, self.key_map, self.E, stream)
        # size phase: counts[(dst, local expert)] -> recv[(src, local expert)]
        send_counts = counts.view(D, El)
        recv_counts = torch.empty_like(send_counts)
        self.transport.all_to_all(recv_counts, send_counts, [1] * D, [1] * D)
        sc = send_counts.cpu()  # the layer's one host sync
        rc = recv_counts.cpu()
        send_rows = sc.sum(1).tolist()
        recv_rows = rc.sum(1).tolist()
        R = int(sum(recv_rows))
        # payload phase
        xp = B.gather(x, order, k, stream)
        xr = torch.empty(R, TD, dtype=x.dtype, device=x.device)
        self.transport.all_to_all(xr, xp, recv_rows, send_rows)
        wr = torch.empty(R, dtype=torch.float32, device=x.device)
        self.transport.all_to_all(wr, wpos, recv_rows, send_rows)
        keys = B.segment_keys(recv_counts.reshape(-1).contiguous(), El, R, stream)
        yr = B.ffn(xr, keys, wr, stream)
        # reverse payload phase and combine at the origin
        yb = torch.empty(S * k, TD, dtype=x.dtype, device=x.device)
        self.transport.all_to_all(yb, yr, send_rows, recv_rows)
        out = B.combine(yb, pos, S, k, stream)
        self.last = {"idx": idx, "w": w, "send_counts": sc, "recv_counts": rc, "recv_rows": R}
        return out


# ------------------------------------------------------------------ exchange over peer memory
class PeerMemoryUnavailable(RuntimeError):
    """Raised on EVERY rank when any rank cannot map its peers' windows (CUDA
    IPC / peer access unavailable), so callers can fall back collectively."""


class PeerExpertParallelMoE:
    """One rank's share of the expert-parallel layer with the exchange done by
    the layer's own kernels through NVLink peer memory (C ABI ``moe_ep_*``,
    csrc/ep_p2p.cu): the count exchange, the gather fused with the payload
    all-to-all, and the return all-to-all fused with the combine.  No NCCL and
    no host synchronisation on the data path, so a forward is one stream-ordered
    call that can be captured in a CUDA graph.

    Same placement and routing as ``ExpertParallelMoE`` (keys = (device, local
    expert), exchange.cpp:95-120 as slot counts); the receive layout is grouped
    by local expert, then source rank, then slot -- the single-GPU order, so
    each row's FFN is the same computation as in ``MoeLayer``.

    ``torch.distributed`` is used only at construction to exchange the
    64-byte CUDA IPC handles of the ranks' windows (any backend).

    ``transport="nccl"`` selects the C ABI's NCCL transport instead
    (csrc/ep_nccl.cu): count all-gather + one host sync + grouped
    ncclSend/ncclRecv of the rows, same routing, FFN and combine; the NCCL
    communicator is created inside the library from a unique id that rank 0
    broadcasts over torch.distributed.
    """

    def __init__(self, ctx, placement: Placement, shape, Wg, W1_local, W2_local, max_tokens: int,
                 rank: int, group=None, max_recv_rows: int = 0, transport: str = "p2p"):
        placement.validate()
        self.ctx, self.lib = ctx, ctx.lib
        self.placement, self.shape, self.rank = placement, shape, rank
        self.D = placement.num_devices
        self.max_tokens = max_tokens
        if transport not in ("p2p", "nccl"):
            raise ValueError("transport must be 'p2p' or 'nccl'")
        self.transport = transport
        d = _capi.EpDesc(rank, self.D, max_tokens, shape.token_dim, shape.hidden_dim,
                         shape.num_experts, shape.top_k, max_recv_rows,
                         _capi.MOE_EP_TRANSPORT_NCCL if transport == "nccl" else _capi.MOE_EP_TRANSPORT_P2P)
        dev_of = np.ascontiguousarray(placement.device_of, dtype=np.int32)
        h = C.c_void_p()
        check(self.lib.moe_ep_create(ctx.h, C.byref(d), _p(Wg), _p(W1_local), _p(W2_local),
                                     dev_of.ctypes.data_as(C.c_void_p), C.byref(h)))
        self.h = h
        self.Wg = Wg  # the gate's TMA descriptor holds Wg's raw pointer
        self.group = group
        if transport == "nccl":
            # the C ABI owns the NCCL communicator; torch.distributed only
            # carries the 128-byte unique id from rank 0
            uid = C.create_string_buffer(_capi.MOE_NCCL_ID_BYTES)
            if rank == 0:
                check(self.lib.moe_nccl_get_unique_id(uid))
            if self.D > 1:
                obj = [bytes(uid.raw)]
                dist.broadcast_object_list(obj, src=0, group=group)
                uid = C.create_string_buffer(obj[0], _capi.MOE_NCCL_ID_BYTES)
            check(self.lib.moe_ep_connect_nccl(self.h, uid))
            return
        buf = C.create_string_buffer(_capi.MOE_EP_HANDLE_BYTES)
        check(self.lib.moe_ep_get_handle(self.h, buf))
        mine = bytes(buf.raw)
        if self.D > 1:
            handles = [None] * self.D
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        st = self.lib.moe_ep_connect(self.h, b"".join(handles))
        err = self.lib.moe_last_error().decode() if st else ""
        if self.D > 1:
            # collective verdict: every rank mapped every peer window, or none proceeds
            ok = torch.tensor([0 if st else 1], dtype=torch.int32,
                              device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if int(ok.item()) == 0:
                self.lib.moe_ep_destroy(self.h)
                self.h = None
                raise PeerMemoryUnavailable(err or "a peer rank could not map the windows")
            dist.barrier(group=group)
        elif st:
            check(st)

    def forward(self, x: torch.Tensor, stream=None, out: torch.Tensor | None = None,
                graph: bool = False) -> torch.Tensor:
        """Collective: every rank calls forward the same number of times."""
        S = x.shape[0]
        if out is None:
            out = torch.empty_like(x)
        fn = self.lib.moe_ep_forward_graph if graph else self.lib.moe_ep_forward
        check(fn(self.h, _p(x), S, _p(out), _s(stream)))
        return out

    def check_errors(self, stream=None):
        check(self.lib.moe_ep_check_errors(self.h, _s(stream)))

    def enable_timing(self, on: bool = True):
        check(self.lib.moe_ep_enable_timing(self.h, 1 if on else 0))

    def stage_times(self) -> dict:
        """ms per stage of the last eager forward (moe_ep_stage_times)."""
        ms = (C.c_float * _capi.MOE_EP_NUM_STAGES)()
        check(self.lib.moe_ep_stage_times(self.h, ms))
        return dict(zip(_capi.EP_STAGES, [float(v) for v in ms]))

    def view(self, S: int) -> dict:
        """Device buffers of the last forward (copies), for parity tests."""
        from .layer import _from_ptr

        v = _capi.EpView()
        check(self.lib.moe_ep_get_view(self.h, C.byref(v)))
        E, k, TD = self.shape.num_experts, self.shape.top_k, self.shape.token_dim
        dev = torch.device("cuda", self.ctx.device)
        ca = _from_ptr(v.counts_all, self.D * E, torch.int32, dev).view(self.D, E)
        El = E // self.D
        R = int(ca[:, self.rank * El:(self.rank + 1) * El].sum())
        R_stored = min(R, int(v.max_recv_rows))  # rows past the receive capacity were never stored
        out = {
            "idx": _from_ptr(v.idx, S * k, torch.int32, dev).view(S, k),
            "w": _from_ptr(v.w, S * k, torch.float32, dev).view(S, k),
            "counts": _from_ptr(v.counts, E, torch.int32, dev),
            "counts_all": ca,
            "dest": _from_ptr(v.dest, S * k, torch.int32, dev),
            "order": _from_ptr(v.order, S * k, torch.int32, dev),
            "n_items": int(_from_ptr(v.n_items, 1, torch.int32, dev)[0]),
            "recv_rows": R,
        }
        if R_stored:
            out["recv_x"] = _from_ptr(v.recv_x, R_stored * TD, torch.bfloat16, dev).view(R_stored, TD)
            out["recv_y"] = _from_ptr(v.recv_y, R_stored * TD, torch.bfloat16, dev).view(R_stored, TD)
            out["recv_w"] = _from_ptr(v.recv_w, R_stored, torch.float32, dev)
        return out

    def close(self):
        if getattr(self, "h", None):
            if self.D > 1 and dist.is_initialized():
                dist.barrier(group=self.group)  # no peer still maps our window
            self.lib.moe_ep_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.moe_ep_destroy(self.h)
                self.h = None
        except Exception:
            pass


def recv_layout(counts_all: np.ndarray, rank: int, El: int):
    """Receive-side row layout of device ``rank`` (host restatement of
    ep_dispatch_kernel's destination rows, for tests): returns
    start[src, local_expert] -- rows are grouped by local expert, then by
    source rank, then in the source's slot order."""
    D = counts_all.shape[0]
    c = counts_all[:, rank * El:(rank + 1) * El].astype(np.int64)  # [src, e]
    col = c.sum(0)
    base = np.concatenate([[0], np.cumsum(col)[:-1]])
    below = np.cumsum(c, axis=0) - c
    return base[None, :] + below
