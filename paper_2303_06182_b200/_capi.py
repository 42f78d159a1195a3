"""ctypes binding of the C ABI declared in include/moe_capi.h.

The shared library ``libmoe_b200.so`` (sm_100a kernels + C ABI) is built
in-tree by ``__graft_entry__.build()``.  There is no CPU fallback: if the
library is missing, or no B200 is present, every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOE_LIB_PATH") or os.path.join(_HERE, "libmoe_b200.so")  # override: A/B builds

MOE_OK = 0
MOE_ERR_INVALID_ARGUMENT = 1
MOE_ERR_CUDA = 2
MOE_ERR_UNSUPPORTED = 3
MOE_ERR_OUT_OF_MEMORY = 4
MOE_ERR_EXPERT_RANGE = 5
MOE_ERR_PEER_TIMEOUT = 6
MOE_EP_MAX_RANKS = 8
MOE_EP_HANDLE_BYTES = 64
MOE_NCCL_ID_BYTES = 128
MOE_EP_TRANSPORT_P2P = 0
MOE_EP_TRANSPORT_NCCL = 1
MOE_EP_NUM_STAGES = 7
EP_STAGES = ["gate_route", "publish", "dispatch", "recv", "ffn", "done", "combine"]

MOE_GATING_STATIC = 0
MOE_GATING_DYNAMIC = 1

# Every symbol include/moe_capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "moe_version", "moe_status_string", "moe_last_error", "moe_ctx_create", "moe_ctx_destroy",
    "moe_ctx_sm_count", "moe_expert_capacity", "moe_dynamic_dispatch_host",
    "moe_static_dispatch_host", "moe_inverse_order_host", "moe_route_dynamic", "moe_route_static",
    "moe_check_errors", "moe_gate_topk", "moe_gather_rows", "moe_combine", "moe_fill_uniform_bf16",
    "moe_layer_create", "moe_layer_destroy", "moe_layer_forward", "moe_layer_forward_graph",
    "moe_layer_forward_host", "moe_layer_get_view", "moe_layer_set_weight_pool",
    "moe_exchange_counts_host", "moe_layer_enable_timing", "moe_layer_stage_times",
    "moe_ffn_create", "moe_ffn_destroy", "moe_ffn_forward", "moe_route_dynamic_keyed",
    "moe_fill_segments", "moe_cache_create", "moe_cache_destroy", "moe_cache_forward",
    "moe_cache_forward_routed", "moe_cache_stats", "moe_cache_resident", "moe_layer_forward_routed",
    "moe_device_alloc", "moe_device_free", "moe_host_alloc", "moe_host_free", "moe_memcpy",
    "moe_stream_create", "moe_stream_destroy", "moe_stream_synchronize",
    "moe_layer_forward_host_batches", "moe_layer_repack",
    "moe_ep_create", "moe_ep_destroy", "moe_ep_get_handle", "moe_ep_connect", "moe_ep_forward",
    "moe_ep_forward_graph", "moe_ep_check_errors", "moe_ep_get_view", "moe_ep_enable_timing",
    "moe_ep_stage_times", "moe_cache_policy_access", "moe_nccl_get_unique_id", "moe_ep_connect_nccl",
    "moe_pack_expert_weights",
]


class MoeError(RuntimeError):
    """A non-OK status from the C ABI."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} [status {status}]")
        self.status = status
        self.msg = msg


class MoeInvalidArgument(MoeError, ValueError):
    """MOE_ERR_INVALID_ARGUMENT -- the reference's std::invalid_argument."""


class LayerDesc(C.Structure):
    _fields_ = [
        ("max_tokens", C.c_int), ("token_dim", C.c_int), ("hidden_dim", C.c_int),
        ("num_experts", C.c_int), ("top_k", C.c_int), ("mode", C.c_int),
        ("capacity_factor", C.c_double), ("tile_n", C.c_int), ("keep_logits", C.c_int),
        ("fuse_combine", C.c_int), ("split_ffn", C.c_int),
        ("keep_layout", C.c_int), ("weights_packed", C.c_int),
    ]


class FfnDesc(C.Structure):
    _fields_ = [("max_rows", C.c_int), ("token_dim", C.c_int), ("hidden_dim", C.c_int),
                ("num_experts", C.c_int), ("tile_n", C.c_int)]


class LayerView(C.Structure):
    _fields_ = [
        ("idx", C.c_void_p), ("w", C.c_void_p), ("logits", C.c_void_p), ("counts", C.c_void_p),
        ("splits", C.c_void_p), ("order", C.c_void_p), ("pos", C.c_void_p),
        ("dropped", C.c_void_p), ("n_dropped", C.c_void_p), ("xp", C.c_void_p),
        ("h", C.c_void_p), ("yw", C.c_void_p), ("n_items", C.c_void_p), ("rows", C.c_int),
        ("capacity", C.c_int), ("tile_n", C.c_int), ("ffn_kernel", C.c_int),
    ]


class EpDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("world_size", C.c_int), ("max_tokens", C.c_int),
                ("token_dim", C.c_int), ("hidden_dim", C.c_int), ("num_experts", C.c_int),
                ("top_k", C.c_int), ("max_recv_rows", C.c_int), ("transport", C.c_int)]


class EpView(C.Structure):
    _fields_ = [
        ("idx", C.c_void_p), ("w", C.c_void_p), ("counts", C.c_void_p), ("counts_all", C.c_void_p),
        ("dest", C.c_void_p), ("order", C.c_void_p), ("recv_x", C.c_void_p), ("recv_y", C.c_void_p),
        ("recv_w", C.c_void_p), ("n_items", C.c_void_p), ("max_recv_rows", C.c_int),
    ]


_lib = None


def _sig(fn, res, *args):
    fn.restype = res
    fn.argtypes = list(args)


def load(path: str = LIB_PATH):
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built -- run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    I, P, D, I64, U64, F = C.c_int, C.c_void_p, C.c_double, C.c_int64, C.c_uint64, C.c_float
    _sig(lib.moe_version, I)
    _sig(lib.moe_status_string, C.c_char_p, I)
    _sig(lib.moe_last_error, C.c_char_p)
    _sig(lib.moe_ctx_create, I, I, C.POINTER(P))
    _sig(lib.moe_ctx_destroy, I, P)
    _sig(lib.moe_ctx_sm_count, I, P)
    _sig(lib.moe_expert_capacity, I, D, I)
    _sig(lib.moe_dynamic_dispatch_host, I, P, P, I, I, I, P, P, P)
    _sig(lib.moe_static_dispatch_host, I, P, P, I, I, I, D, P, P, I64, P, P)
    _sig(lib.moe_inverse_order_host, I, P, P, I64, P, I64)
    _sig(lib.moe_route_dynamic, I, P, P, I, I, I, P, P, P, P, P)
    _sig(lib.moe_route_static, I, P, P, I, I, I, I, P, P, P, P, P, P)
    _sig(lib.moe_check_errors, I, P, P)
    _sig(lib.moe_gate_topk, I, P, P, P, I, I, I, I, P, P, P, P)
    _sig(lib.moe_gather_rows, I, P, P, P, I, I, I, P, P)
    _sig(lib.moe_combine, I, P, P, P, I, I, I, P, P)
    _sig(lib.moe_fill_uniform_bf16, I, P, P, I64, U64, U64, F, P)
    _sig(lib.moe_layer_create, I, P, C.POINTER(LayerDesc), P, P, P, C.POINTER(P))
    _sig(lib.moe_layer_destroy, I, P)
    _sig(lib.moe_layer_forward, I, P, P, I, P, P)
    _sig(lib.moe_layer_forward_graph, I, P, P, I, P, P)
    _sig(lib.moe_layer_forward_host, I, P, P, I, P, P)
    _sig(lib.moe_layer_forward_host_batches, I, P, P, P, P, I, P)
    _sig(lib.moe_layer_repack, I, P, P)
    _sig(lib.moe_pack_expert_weights, I, P, P, P, I64, I, P)
    _sig(lib.moe_layer_get_view, I, P, C.POINTER(LayerView))
    _sig(lib.moe_layer_set_weight_pool, I, P, P, P, I, P)
    _sig(lib.moe_exchange_counts_host, I, P, P, I, I, I, P, I, I, P)
    _sig(lib.moe_layer_enable_timing, I, P, I)
    _sig(lib.moe_layer_stage_times, I, P, I, P)
    _sig(lib.moe_ffn_create, I, P, C.POINTER(FfnDesc), P, P, C.POINTER(P))
    _sig(lib.moe_ffn_destroy, I, P)
    _sig(lib.moe_ffn_forward, I, P, P, P, P, I, P, P)
    _sig(lib.moe_route_dynamic_keyed, I, P, P, I, I, I, P, I, P, P, P, P, P, P, P)
    _sig(lib.moe_fill_segments, I, P, P, I, I, P, P)
    _sig(lib.moe_cache_create, I, P, P, P, I, I, C.POINTER(P))
    _sig(lib.moe_cache_destroy, I, P)
    _sig(lib.moe_cache_forward, I, P, P, I, P, P)
    _sig(lib.moe_cache_forward_routed, I, P, P, P, P, I, P, P)
    _sig(lib.moe_cache_stats, I, P, P, P)
    _sig(lib.moe_cache_resident, I, P, P, P)
    _sig(lib.moe_cache_policy_access, I, P, P, I, I, P, I, P, C.c_int64, P)
    _sig(lib.moe_layer_forward_routed, I, P, P, P, P, I, P, P)
    if not hasattr(lib, "moe_ep_create"):  # an older build (A/B runs via MOE_LIB_PATH)
        _lib = lib
        return lib
    _sig(lib.moe_ep_create, I, P, C.POINTER(EpDesc), P, P, P, P, C.POINTER(P))
    _sig(lib.moe_ep_destroy, I, P)
    _sig(lib.moe_ep_get_handle, I, P, P)
    _sig(lib.moe_ep_connect, I, P, P)
    _sig(lib.moe_ep_forward, I, P, P, I, P, P)
    _sig(lib.moe_ep_forward_graph, I, P, P, I, P, P)
    _sig(lib.moe_ep_check_errors, I, P, P)
    _sig(lib.moe_ep_get_view, I, P, C.POINTER(EpView))
    _sig(lib.moe_ep_enable_timing, I, P, I)
    _sig(lib.moe_ep_stage_times, I, P, P)
    _sig(lib.moe_nccl_get_unique_id, I, P)
    _sig(lib.moe_ep_connect_nccl, I, P, P)
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == MOE_OK:
        return
    msg = load().moe_last_error().decode()
    if status == MOE_ERR_INVALID_ARGUMENT:
        raise MoeInvalidArgument(status, msg)
    raise MoeError(status, msg)
