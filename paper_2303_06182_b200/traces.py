"""Routing workloads for the GPU layer: the reference's synthetic skewed trace
generator (include/moesim/trace.hpp gen_synthetic_trace, implemented in C++ in
libmoesim_b200.so) as numpy arrays ready for moe_layer_forward_routed /
moe_cache_forward_routed."""
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
    return _LIB


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
