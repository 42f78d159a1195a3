"""Routing workloads for the GPU layer: the reference's synthetic skewed trace
generator (include/moesim/trace.hpp gen_synthetic_trace, implemented in C++ in
libmoesim_b200.so) as numpy arrays ready for moe_layer_forward_routed /
moe_cache_forward_routed, and the reference's JSON Lines trace files
(include/moesim/trace.hpp load_token_trace / save_token_trace)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._capi import load

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        load()
        _LIB = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmoesim_b200.so"))
        f = _LIB.moesim_gen_synthetic_routing
        f.restype = C.c_int
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                      C.c_void_p, C.c_void_p, C.c_char_p, C.c_int]
        f = _LIB.moesim_save_synthetic_trace
        f.restype = C.c_int
        f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                      C.c_char_p, C.c_char_p, C.c_int]
        f = _LIB.moesim_trace_roundtrip
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, C.c_char_p, C.c_void_p, C.c_char_p, C.c_int]
        f = _LIB.moesim_trace_loads
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_char_p, C.c_int]
    return _LIB


def _raise(rc: int, err) -> None:
    if rc == 1:
        raise ValueError(err.value.decode())
    if rc:
        raise RuntimeError(err.value.decode())


def save_synthetic_trace(path, E: int, k: int, batches: int, S: int, zipf_skew: float = 1.2,
                         persistence: float = 0.9, active_fraction: float = 1.0, seed: int = 0) -> None:
    """Generate a synthetic trace and write it as JSON Lines (reference format)."""
    err = C.create_string_buffer(512)
    _raise(_lib().moesim_save_synthetic_trace(E, k, batches, S, zipf_skew, persistence, active_fraction,
                                              seed, str(path).encode(), err, 512), err)


def trace_roundtrip(in_path, out_path="") -> tuple[int, int, int]:
    """Load (validating) a trace file; re-save it to out_path if given.
    Returns (num_experts, top_k, num_batches)."""
    dims = np.zeros(3, np.int32)
    err = C.create_string_buffer(1024)
    _raise(_lib().moesim_trace_roundtrip(str(in_path).encode(), str(out_path).encode(),
                                         dims.ctypes.data_as(C.c_void_p), err, 1024), err)
    return tuple(int(v) for v in dims)


def trace_loads(path, E: int, B: int) -> np.ndarray:
    """Load matrix share [E, B] of a trace file (columns sum to 1)."""
    share = np.zeros(E * B, np.float64)
    err = C.create_string_buffer(1024)
    _raise(_lib().moesim_trace_loads(str(path).encode(), share.ctypes.data_as(C.c_void_p), E * B, err,
                                     1024), err)
    return share.reshape(B, E).T


def skewed_routing(E: int, k: int, batches: int, S: int, zipf_skew: float = 1.2, persistence: float = 0.9,
                   active_fraction: float = 1.0, seed: int = 0):
    """experts int32 [batches, S, k], weights float64 [batches, S, k]."""
    ex = np.zeros(batches * S * k, np.int32)
    w = np.zeros(batches * S * k, np.float64)
    err = C.create_string_buffer(256)
    rc = _lib().moesim_gen_synthetic_routing(E, k, batches, S, zipf_skew, persistence, active_fraction, seed,
                                             ex.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), err, 256)
    if rc:
        raise ValueError(err.value.decode())
    return ex.reshape(batches, S, k), w.reshape(batches, S, k)
