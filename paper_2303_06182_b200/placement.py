"""Host placement policy for expert parallelism, from the C++ library.

The policies live in ``libmoesim_b200.so`` (paper_2303_06182_b200/host/
balance.cpp, the drop-in of the reference's proj/src/balance.cpp:59-165) and
are bound here through the C entry points of include/moesim/placement_c.h,
so Python and C++ hosts place experts with the same code.  Histories are
E x B load-share matrices (LoadMatrix::share).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
CXX_PATH = os.path.join(_HERE, "libmoesim_b200.so")
_cxx = None


class PlacementError(ValueError):
    pass


def load_cxx():
    global _cxx
    if _cxx is None:
        if not os.path.exists(CXX_PATH):
            raise ImportError(f"{CXX_PATH} not built -- run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(CXX_PATH)
        I, P, D = C.c_int, C.c_void_p, C.c_double
        lib.moesim_placement_last_error.restype = C.c_char_p
        lib.moesim_placement_last_error.argtypes = []
        for name, args in (("moesim_contiguous_place", [I, I, P]),
                           ("moesim_greedy_place", [P, I, I, I, P]),
                           ("moesim_anticorr_place", [P, I, I, I, D, P]),
                           ("moesim_pearson_corr", [P, I, I, P]),
                           ("moesim_eval_balance", [P, I, I, P, I, P, P, P, P])):
            fn = getattr(lib, name)
            fn.restype = I
            fn.argtypes = args
        _cxx = lib
    return _cxx


def _ok(rc: int):
    if rc:
        raise PlacementError(load_cxx().moesim_placement_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _history(loads):
    h = np.ascontiguousarray(loads, dtype=np.float64)
    if h.ndim != 2:
        raise PlacementError("load history must be an E x B matrix")
    return h


def contiguous_place(E: int, D: int) -> np.ndarray:
    out = np.zeros(E, np.int32)
    _ok(load_cxx().moesim_contiguous_place(E, D, _ptr(out)))
    return out


def greedy_place(loads, D: int) -> np.ndarray:
    h = _history(loads)
    out = np.zeros(h.shape[0], np.int32)
    _ok(load_cxx().moesim_greedy_place(_ptr(h), h.shape[0], h.shape[1], D, _ptr(out)))
    return out


def anticorr_place(loads, D: int, weight: float = 0.5) -> np.ndarray:
    h = _history(loads)
    out = np.zeros(h.shape[0], np.int32)
    _ok(load_cxx().moesim_anticorr_place(_ptr(h), h.shape[0], h.shape[1], D, float(weight), _ptr(out)))
    return out


def pearson_corr(loads) -> np.ndarray:
    h = _history(loads)
    out = np.zeros((h.shape[0], h.shape[0]), np.float64)
    _ok(load_cxx().moesim_pearson_corr(_ptr(h), h.shape[0], h.shape[1], _ptr(out)))
    return out


def eval_balance(device_of, D: int, loads) -> dict:
    """BalanceReport of balance.hpp: per-batch device load shares, Max Load,
    Avg Max Load and the max deviation from 1/D."""
    h = _history(loads)
    dev = np.ascontiguousarray(device_of, dtype=np.int32)
    dl = np.zeros((D, h.shape[1]), np.float64)
    m, a, o = C.c_double(), C.c_double(), C.c_double()
    _ok(load_cxx().moesim_eval_balance(_ptr(dev), dev.size, D, _ptr(h), h.shape[1], _ptr(dl), C.byref(m),
                                       C.byref(a), C.byref(o)))
    return {"device_load": dl, "max_load": m.value, "avg_max_load": a.value, "objective": o.value}
