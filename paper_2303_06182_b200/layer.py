"""Device-resident MoE layer over the C ABI (include/moe_capi.h).

``MoeLayer`` is the perf path: torch owns the device memory (weights, inputs,
outputs) and streams; every byte of arithmetic runs in the sm_100a kernels of
``libmoe_b200.so`` (gate, route, gather, grouped FFN, combine).  There is no
torch / CPU compute path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _capi
from ._capi import check, load

SEED = 2303061820


class Context:
    """One moe_ctx per device (the library handle)."""

    _by_device: dict = {}

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = C.c_void_p()
        check(self.lib.moe_ctx_create(device, C.byref(h)))
        self.h = h

    @classmethod
    def get(cls, device: int | None = None) -> "Context":
        if device is None:
            device = torch.cuda.current_device()
        if device not in cls._by_device:
            cls._by_device[device] = Context(device)
        return cls._by_device[device]

    @classmethod
    def close_all(cls):
        """Destroy every cached context (tools / sanitizer runs: no live
        layer may still use them)."""
        for c in cls._by_device.values():
            c.lib.moe_ctx_destroy(c.h)
        cls._by_device.clear()

    @property
    def sm_count(self) -> int:
        return self.lib.moe_ctx_sm_count(self.h)


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _p(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def fill_uniform_bf16(t: torch.Tensor, seed: int, tensor_id: int, scale: float, ctx=None, stream=None):
    """Counter-based synthetic bf16 (bit-identical to oracle.layer.synth_bf16)."""
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
    ctx = ctx or Context.get(t.device.index)
    check(ctx.lib.moe_fill_uniform_bf16(ctx.h, _p(t), t.numel(), seed, tensor_id, float(scale),
                                        _stream_ptr(stream)))
    return t


@dataclass
class LayerShape:
    """The paper's MoE layer shape: TD, HD, E, top-k."""

    token_dim: int
    hidden_dim: int
    num_experts: int
    top_k: int


class MoeLayer:
    """One MoE layer (gate -> dispatch -> expert FFN -> combine) on a B200.

    Weights (bf16, caller-visible torch tensors): Wg [E,TD], W1 [E,HD,TD],
    W2 [E,TD,HD].  ``mode`` is "dynamic" (the paper's dynamic gating, the
    product path) or "static" (capacity-factor comparison mode).
    """

    def __init__(self, shape: LayerShape, max_tokens: int, mode: str = "dynamic",
                 capacity_factor: float = 1.0, weights=None, keep_logits: bool = False,
                 tile_n: int = 0, device: int | None = None, seed: int = SEED, fuse_combine: bool = False,
                 split_ffn: bool = False, keep_layout: bool = False,
                 pack_in_place: bool = False, pool_only: bool = False):
        """pack_in_place: the caller's W1/W2 tensors are repacked IN PLACE into
        the tile layout the fused FFN streams and the layer keeps no copy
        (expert weights held once; the tensors are no longer row-major
        afterwards).  pool_only: no expert weights on the device (W1/W2 may
        be None) -- attach an ExpertCache before forwarding."""
        self.ctx = Context.get(device)
        dev = torch.device("cuda", self.ctx.device)
        TD, HD, E, k = shape.token_dim, shape.hidden_dim, shape.num_experts, shape.top_k
        self.shape = shape
        self.mode = mode
        self.capacity_factor = capacity_factor
        self.max_tokens = max_tokens
        if weights is None:
            weights = make_weights(shape, ctx=self.ctx, seed=seed)
        self.Wg, self.W1, self.W2 = weights
        if pool_only:
            self.W1 = self.W2 = None
        for t, sh in ((self.Wg, (E, TD)), (self.W1, (E, HD, TD)), (self.W2, (E, TD, HD))):
            if t is None:
                continue
            assert t.dtype == torch.bfloat16 and t.is_contiguous() and tuple(t.shape) == sh, sh
            assert t.device == dev
        self.weights_packed = bool(pack_in_place) and not pool_only
        if self.weights_packed:
            pack_expert_weights_(self.W1, self.ctx)
            pack_expert_weights_(self.W2, self.ctx)
        d = _capi.LayerDesc(max_tokens, TD, HD, E, k,
                            _capi.MOE_GATING_DYNAMIC if mode == "dynamic" else _capi.MOE_GATING_STATIC,
                            float(capacity_factor), int(tile_n), int(bool(keep_logits)), int(bool(fuse_combine)),
                            int(bool(split_ffn)), int(bool(keep_layout)),
                            int(self.weights_packed))
        h = C.c_void_p()
        check(self.ctx.lib.moe_layer_create(self.ctx.h, C.byref(d), _p(self.Wg), _p(self.W1),
                                            _p(self.W2), C.byref(h)))
        self.h = h

    def repack(self, stream=None):
        """Refresh the layer's packed copy of W1/W2 after in-place weight updates."""
        check(self.ctx.lib.moe_layer_repack(self.h, _stream_ptr(stream)))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.moe_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, graph: bool = False,
                stream=None) -> torch.Tensor:
        assert x.dtype == torch.bfloat16 and x.is_contiguous() and x.shape[1] == self.shape.token_dim
        if out is None:
            out = torch.empty_like(x)
        fn = self.ctx.lib.moe_layer_forward_graph if graph else self.ctx.lib.moe_layer_forward
        check(fn(self.h, _p(x), x.shape[0], _p(out), _stream_ptr(stream)))
        return out

    __call__ = forward

    def forward_routed(self, x: torch.Tensor, idx: torch.Tensor, w: torch.Tensor,
                       out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Forward with caller-provided routing (idx [S,k] int32, w [S,k] fp32
        on the device) instead of the gate -- trace replay / skewed workloads."""
        assert idx.dtype == torch.int32 and w.dtype == torch.float32 and idx.shape == w.shape
        if out is None:
            out = torch.empty_like(x)
        check(self.ctx.lib.moe_layer_forward_routed(self.h, _p(x), _p(idx.contiguous()), _p(w.contiguous()),
                                                     x.shape[0], _p(out), _stream_ptr(stream)))
        return out

    def forward_host(self, x_host: torch.Tensor, out_host: torch.Tensor, stream=None):
        """End-to-end: pinned host bf16 in -> pinned host bf16 out (copies inside)."""
        check(self.ctx.lib.moe_layer_forward_host(self.h, _p(x_host), x_host.shape[0], _p(out_host),
                                                  _stream_ptr(stream)))
        return out_host

    def forward_host_batches(self, xs_host, outs_host, stream):
        """Pipelined end-to-end path over a queue of batches: pinned host bf16
        in -> pinned host bf16 out for every batch, uploads and read-backs
        overlapped with the neighbouring batches' compute (moe_capi.h)."""
        n = len(xs_host)
        if len(outs_host) != n:
            raise ValueError("one output buffer per batch")
        xp = (C.c_void_p * n)(*[x.data_ptr() for x in xs_host])
        op = (C.c_void_p * n)(*[o.data_ptr() for o in outs_host])
        sz = (C.c_int * n)(*[x.shape[0] for x in xs_host])
        check(self.ctx.lib.moe_layer_forward_host_batches(self.h, xp, sz, op, n,
                                                          _stream_ptr(stream)))
        return outs_host

    def check_errors(self, stream=None):
        check(self.ctx.lib.moe_check_errors(self.ctx.h, _stream_ptr(stream)))

    def view(self) -> dict:
        """Internal device buffers of the last forward, as torch tensors."""
        v = _capi.LayerView()
        check(self.ctx.lib.moe_layer_get_view(self.h, C.byref(v)))
        E, k, TD, HD = (self.shape.num_experts, self.shape.top_k, self.shape.token_dim,
                        self.shape.hidden_dim)
        S = self.max_tokens
        dev = torch.device("cuda", self.ctx.device)

        def wrap(ptr, n, dtype):
            if not ptr or n <= 0:
                return None
            return _from_ptr(ptr, n, dtype, dev)

        rows = v.rows
        out = {
            "idx": wrap(v.idx, S * k, torch.int32), "w": wrap(v.w, S * k, torch.float32),
            "logits": wrap(v.logits, S * E, torch.float32), "counts": wrap(v.counts, E, torch.int32),
            "splits": wrap(v.splits, E + 1, torch.int32), "order": wrap(v.order, rows, torch.int32),
            "pos": wrap(v.pos, S * k, torch.int32), "n_items": wrap(v.n_items, 1, torch.int32),
            "xp": wrap(v.xp, rows * TD, torch.bfloat16), "h": wrap(v.h, rows * HD, torch.bfloat16),
            "yw": wrap(v.yw, rows * TD, torch.bfloat16), "rows": rows, "capacity": v.capacity,
            "tile_n": v.tile_n, "ffn_kernel": v.ffn_kernel,
        }
        if v.dropped:
            out["dropped"] = wrap(v.dropped, 2 * S * k, torch.int32)
            out["n_dropped"] = wrap(v.n_dropped, 1, torch.int32)
        return out


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        load()  # libmoe_b200.so pulls libcudart.so.12 into the process
        _CUDART = C.CDLL("libcudart.so.12")
        _CUDART.cudaMemcpy.restype = C.c_int
        _CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    return _CUDART


def _from_ptr(ptr: int, n: int, dtype, device) -> torch.Tensor:
    """Device-to-device copy of n elements of library-owned memory into a
    fresh torch tensor (so the result outlives the layer)."""
    esz = torch.empty((), dtype=dtype).element_size()
    buf = torch.empty(n, dtype=dtype, device=device)
    torch.cuda.current_stream(device).synchronize()
    err = _cudart().cudaMemcpy(C.c_void_p(buf.data_ptr()), C.c_void_p(ptr), C.c_size_t(n * esz),
                               3)  # cudaMemcpyDeviceToDevice
    if int(err) != 0:
        raise RuntimeError(f"cudaMemcpy failed ({err})")
    return buf


def make_weights(shape: LayerShape, device=None, seed: int = SEED, ctx=None):
    """Random-init expert weights with the counter generator (on the GPU).
    std: Wg 1/sqrt(TD), W1 sqrt(2/TD), W2 1/sqrt(HD) (uniform, a = sqrt(3) std)."""
    import math

    ctx = ctx or Context.get(device)
    dev = torch.device("cuda", ctx.device)
    TD, HD, E = shape.token_dim, shape.hidden_dim, shape.num_experts
    r3 = math.sqrt(3.0)
    Wg = torch.empty(E, TD, dtype=torch.bfloat16, device=dev)
    W1 = torch.empty(E, HD, TD, dtype=torch.bfloat16, device=dev)
    W2 = torch.empty(E, TD, HD, dtype=torch.bfloat16, device=dev)
    fill_uniform_bf16(Wg, seed, 2, r3 / math.sqrt(TD), ctx)
    fill_uniform_bf16(W1, seed, 3, r3 * math.sqrt(2.0 / TD), ctx)
    fill_uniform_bf16(W2, seed, 4, r3 / math.sqrt(HD), ctx)
    return Wg, W1, W2


def pack_expert_weights_(W: torch.Tensor, ctx=None, stream=None) -> torch.Tensor:
    """Repack expert weights [E, rows, K] (bf16, device) IN PLACE into the
    tile layout of the fused FFN (moe_pack_expert_weights); returns W."""
    assert W.dtype == torch.bfloat16 and W.is_cuda and W.is_contiguous() and W.dim() == 3
    ctx = ctx or Context.get(W.device.index)
    check(ctx.lib.moe_pack_expert_weights(ctx.h, _p(W), _p(W), W.shape[0] * W.shape[1], W.shape[2],
                                          _stream_ptr(stream)))
    return W


def make_tokens(S: int, TD: int, device=None, seed: int = SEED, ctx=None):
    import math

    ctx = ctx or Context.get(device)
    x = torch.empty(S, TD, dtype=torch.bfloat16, device=torch.device("cuda", ctx.device))
    return fill_uniform_bf16(x, seed, 1, math.sqrt(3.0), ctx)


class ExpertCache:
    """GPU-resident LIFO/FIFO expert cache over pinned host weights
    (moe_cache_*).  While attached, the layer reads its
    expert weights from the cache's slot pool: run forwards through the cache."""

    POLICIES = {"lifo": 0, "fifo": 1}

    def __init__(self, layer: MoeLayer, n_slots: int, policy: str = "lifo", W1_host=None, W2_host=None):
        self.layer = layer
        self.ctx = layer.ctx
        if (W1_host is None or W2_host is None) and (layer.W1 is None or layer.weights_packed):
            raise ValueError("pass the row-major pinned host weights (W1_host, W2_host)")
        self.W1_host = W1_host if W1_host is not None else layer.W1.cpu().pin_memory()
        self.W2_host = W2_host if W2_host is not None else layer.W2.cpu().pin_memory()
        for t in (self.W1_host, self.W2_host):
            assert t.is_pinned() and t.dtype == torch.bfloat16 and t.is_contiguous()
        h = C.c_void_p()
        check(self.ctx.lib.moe_cache_create(layer.h, _p(self.W1_host), _p(self.W2_host), n_slots,
                                            self.POLICIES[policy], C.byref(h)))
        self.h = h
        self.n_slots = n_slots

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.moe_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, x, out=None, stream=None):
        out = torch.empty_like(x) if out is None else out
        check(self.ctx.lib.moe_cache_forward(self.h, _p(x), x.shape[0], _p(out), _stream_ptr(stream)))
        return out

    def forward_routed(self, x, idx, w, out=None, stream=None):
        out = torch.empty_like(x) if out is None else out
        check(self.ctx.lib.moe_cache_forward_routed(self.h, _p(x), _p(idx.contiguous()), _p(w.contiguous()),
                                                    x.shape[0], _p(out), _stream_ptr(stream)))
        return out

    def stats(self) -> dict:
        tot = (C.c_int64 * 5)()
        last = (C.c_int * 5)()
        check(self.ctx.lib.moe_cache_stats(self.h, C.cast(tot, C.c_void_p), C.cast(last, C.c_void_p)))
        keys = ["accesses", "hits", "misses", "evictions"]
        d = {k: int(v) for k, v in zip(keys, tot[:4])}
        d["bytes_copied"] = int(tot[4])
        d["last"] = {k: int(v) for k, v in zip(keys + ["waves"], last[:5])}
        return d

    def resident(self) -> list:
        n = C.c_int(0)
        buf = (C.c_int32 * max(self.n_slots, 1))()
        check(self.ctx.lib.moe_cache_resident(self.h, C.cast(buf, C.c_void_p), C.byref(n)))
        return [int(x) for x in buf[:n.value]]
