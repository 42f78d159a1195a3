"""ctypes bindings for the two native checkers (TEST INFRASTRUCTURE ONLY).

``ref_lib()``   oracle/_ref/libmoesim_ref.so -- the reference compiled verbatim.
``c_oracle()``  oracle/_build/liboracle.so  -- plain-C restatement.

Both are built by ``make -C oracle`` (``__graft_entry__.build()`` runs it).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libmoesim_ref.so")
ORACLE_SO = os.path.join(_HERE, "_build", "liboracle.so")

_I = C.c_int
_D = C.c_double
_P = C.c_void_p
_I64 = C.c_int64

_ref = None
_c = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _sig(fn, res, *args):
    fn.restype = res
    fn.argtypes = list(args)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle` with /root/reference present")
        lib = C.CDLL(REF_SO)
        _sig(lib.ref_last_error, C.c_char_p)
        _sig(lib.ref_expert_capacity, _I, _D, _I)
        _sig(lib.ref_waste_factor, _D, _I, _D, _I)
        _sig(lib.ref_dispatch_mask_elements, _I64, _I, _I, _D)
        _sig(lib.ref_dynamic_dispatch, _I, _P, _P, _I, _I, _I, _I, _P, _P, _P)
        _sig(lib.ref_static_dispatch, _I, _P, _P, _I, _I, _I, _D, _I, _P, _P, _I, _P, _P)
        _sig(lib.ref_combine_dynamic, _I, _P, _P, _I, _I, _I, _P, _I, _P, _P, _P, _P)
        _sig(lib.ref_combine_static, _I, _P, _P, _I, _I, _I, _D, _P, _I, _P, _P, _P, _P)
        _sig(lib.ref_dispatch_cost_counts, _I, _P, _I, _I, _I, _I, _P)
        _sig(lib.ref_debug_json, _I, _P, _I, _I, _I, _D, _I, C.c_char_p, _I)
        _sig(lib.ref_cache_new, _P)
        _sig(lib.ref_cache_free, None, _P)
        _sig(lib.ref_cache_access, _I, _P, _P, _I, _I, _I, _P, _I, _P, _P, _P)
        _sig(lib.ref_greedy_place, _I, _P, _I, _I, _I, _P)
        _sig(lib.ref_contiguous_place, _I, _I, _I, _P)
        _sig(lib.ref_anticorr_place, _I, _P, _I, _I, _I, _D, _P)
        _sig(lib.ref_pearson_corr, _I, _P, _I, _I, _P)
        _sig(lib.ref_eval_balance, _I, _P, _I, _I, _P, _I, _P)
        _sig(lib.ref_plan_dynamic_exchange, _I, _P, _I, _I, _I, _I, _P, _I64, _P, _P)
        _sig(lib.ref_gen_synthetic_trace, _I, _I, _I, _I, _I, _D, _D, _D, C.c_uint64, _P, _P)
        _sig(lib.ref_save_synthetic_trace, _I, _I, _I, _I, _I, _D, _D, _D, C.c_uint64, C.c_char_p)
        _sig(lib.ref_trace_roundtrip, _I, C.c_char_p, C.c_char_p, _P)
        _sig(lib.ref_trace_loads, _I, C.c_char_p, _P, _I)
        _sig(lib.ref_time_routing, _I, _P, _P, _I, _I, _I, _D, _I, _P)
        _ref = lib
    return _ref


def c_oracle():
    global _c
    if _c is None:
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
        lib = C.CDLL(ORACLE_SO)
        _sig(lib.or_last_error, C.c_char_p)
        _sig(lib.or_expert_capacity, _I, _D, _I)
        _sig(lib.or_dynamic_dispatch, _I, _P, _I, _I, _I, _P, _P, _P, _P)
        _sig(lib.or_static_dispatch, _I, _P, _I, _I, _I, _D, _P, _P, _I64, _P, _P, _P)
        _sig(lib.or_combine_positions, _I, _P, _I, _I, _P)
        _sig(lib.or_waste_factor, _D, _I, _D, _I)
        _sig(lib.or_dispatch_mask_elements, _I64, _I, _I, _D)
        _sig(lib.or_exchange_counts, _I, _P, _I, _I, _I, _P, _P)
        _c = lib
    return _c


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(ValueError):
    pass


# --------------------------------------------------------------- reference
def ref_dynamic_dispatch(experts: np.ndarray, E: int, weights=None, mode_static=False):
    """proj/src/gating.cpp:58-86 via the verbatim build. experts: [S, k] int."""
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    order = np.zeros(max(S * k, 1), np.int32)
    counts = np.zeros(max(E, 1), np.int32)
    splits = np.zeros(max(E + 1, 1), np.int32)
    rc = ref_lib().ref_dynamic_dispatch(_ptr(ex), None if w is None else _ptr(w), S, k, E,
                                        int(mode_static), _ptr(order), _ptr(counts), _ptr(splits))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return order[:S * k], counts[:E], splits[:E + 1]


def ref_time_routing(experts: np.ndarray, weights: np.ndarray, E: int, C_: float = 0.0, reps: int = 5):
    """The reference's routing functions on one thread, Batch prebuilt (no
    marshalling in the timed region); best of ``reps`` seconds per call."""
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    wt = np.ascontiguousarray(weights, dtype=np.float64)
    sec = np.zeros(4, np.float64)
    if ref_lib().ref_time_routing(_ptr(ex), _ptr(wt), S, k, E, float(C_), reps, _ptr(sec)):
        raise OracleError(ref_lib().ref_last_error().decode())
    out = {"dynamic_dispatch": sec[0], "combine_dynamic": sec[1]}
    if C_ > 0:
        out.update({"static_dispatch": sec[2], "combine_static": sec[3]})
    return out


def ref_static_dispatch(experts: np.ndarray, E: int, C_: float, weights=None, mode_static=True):
    """proj/src/gating.cpp:30-56 -> (capacity, slots [E, cap], dropped [n, 2])."""
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    cap_guess = max(1, ref_lib().ref_expert_capacity(C_, S)) if C_ > 0 else 1
    slots = np.zeros(max(E, 1) * cap_guess, np.int32)
    dropped = np.zeros(2 * S * k + 2, np.int32)
    cap = C.c_int(0)
    nd = C.c_int(0)
    rc = ref_lib().ref_static_dispatch(_ptr(ex), None if w is None else _ptr(w), S, k, E, C_,
                                       int(mode_static), C.byref(cap), _ptr(slots), slots.size,
                                       _ptr(dropped), C.byref(nd))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    c = cap.value
    return c, slots[:E * c].reshape(E, c), dropped[:2 * nd.value].reshape(-1, 2)


def ref_combine_dynamic(experts, weights, E, payload):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    w = np.ascontiguousarray(weights, dtype=np.float64)
    pl = np.ascontiguousarray(payload, dtype=np.int32)
    n = np.zeros(S, np.int32)
    oe = np.zeros(S * k, np.int32)
    ow = np.zeros(S * k, np.float64)
    op = np.zeros(S * k, np.int32)
    rc = ref_lib().ref_combine_dynamic(_ptr(ex), _ptr(w), S, k, E, _ptr(pl), pl.size, _ptr(n),
                                       _ptr(oe), _ptr(ow), _ptr(op))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return n, oe.reshape(S, k), ow.reshape(S, k), op.reshape(S, k)


def ref_combine_static(experts, weights, E, C_, payload):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    w = np.ascontiguousarray(weights, dtype=np.float64)
    pl = np.ascontiguousarray(payload, dtype=np.int32)
    n = np.zeros(S, np.int32)
    oe = np.zeros(S * k, np.int32)
    ow = np.zeros(S * k, np.float64)
    op = np.zeros(S * k, np.int32)
    rc = ref_lib().ref_combine_static(_ptr(ex), _ptr(w), S, k, E, C_, _ptr(pl), pl.size, _ptr(n),
                                      _ptr(oe), _ptr(ow), _ptr(op))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return n, oe.reshape(S, k), ow.reshape(S, k), op.reshape(S, k)


def ref_debug_json(experts, E, C_=0.0, is_static=False) -> str:
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    buf = C.create_string_buffer(1 << 20)
    rc = ref_lib().ref_debug_json(_ptr(ex), S, k, E, C_, int(is_static), buf, len(buf))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return buf.value.decode()


def ref_dispatch_cost_counts(experts, E, token_dim):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    out = np.zeros(3, np.int64)
    rc = ref_lib().ref_dispatch_cost_counts(_ptr(ex), S, k, E, token_dim, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return tuple(int(x) for x in out)


class RefCache:
    """buffer.cpp:57-130 access_batch on a CacheState handle."""

    def __init__(self):
        self.h = ref_lib().ref_cache_new()

    def __del__(self):
        try:
            ref_lib().ref_cache_free(self.h)
        except Exception:
            pass

    def access(self, active, cache_size, policy=0, future=None):
        a = np.ascontiguousarray(active, dtype=np.int32)
        f = None if future is None else np.ascontiguousarray(future, dtype=np.int32)
        stats = np.zeros(4, np.int32)
        res = np.zeros(max(cache_size, 1) + 1, np.int32)
        nres = C.c_int(0)
        rc = ref_lib().ref_cache_access(self.h, _ptr(a), a.size, cache_size, policy,
                                        None if f is None else _ptr(f), 0 if f is None else f.size,
                                        _ptr(stats), _ptr(res), C.byref(nres))
        if rc:
            raise OracleError(ref_lib().ref_last_error().decode())
        return tuple(int(x) for x in stats), [int(x) for x in res[:nres.value]]


def ref_greedy_place(loads: np.ndarray, D: int):
    l = np.ascontiguousarray(loads, dtype=np.float64)
    E, B = l.shape
    out = np.zeros(E, np.int32)
    rc = ref_lib().ref_greedy_place(_ptr(l), E, B, D, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return out


def ref_contiguous_place(E: int, D: int):
    out = np.zeros(E, np.int32)
    rc = ref_lib().ref_contiguous_place(E, D, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return out


def _loads(loads):
    l = np.ascontiguousarray(loads, dtype=np.float64)
    return l, l.shape[0], l.shape[1]


def ref_anticorr_place(loads: np.ndarray, D: int, weight: float = 0.5):
    l, E, B = _loads(loads)
    out = np.zeros(E, np.int32)
    rc = ref_lib().ref_anticorr_place(_ptr(l), E, B, D, weight, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return out


def ref_pearson_corr(loads: np.ndarray):
    l, E, B = _loads(loads)
    out = np.zeros((E, E), np.float64)
    rc = ref_lib().ref_pearson_corr(_ptr(l), E, B, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return out


def ref_eval_balance(device_of, D: int, loads: np.ndarray):
    """(max_load, avg_max_load, objective) of balance.cpp:153-165."""
    l, E, B = _loads(loads)
    dev = np.ascontiguousarray(device_of, dtype=np.int32)
    out = np.zeros(3, np.float64)
    rc = ref_lib().ref_eval_balance(_ptr(dev), E, D, _ptr(l), B, _ptr(out))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return tuple(float(x) for x in out)


def ref_plan_dynamic_exchange(experts, E, D, device_of, token_bytes):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    dev = np.ascontiguousarray(device_of, dtype=np.int32)
    size_b = np.zeros(D * D, np.int64)
    pay_b = np.zeros(D * D, np.int64)
    rc = ref_lib().ref_plan_dynamic_exchange(_ptr(ex), S, k, E, D, _ptr(dev), token_bytes,
                                             _ptr(size_b), _ptr(pay_b))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return size_b.reshape(D, D), pay_b.reshape(D, D)


def ref_gen_synthetic_trace(E, k, B, S, skew, persistence, active_fraction, seed):
    experts = np.zeros(B * S * k, np.int32)
    weights = np.zeros(B * S * k, np.float64)
    rc = ref_lib().ref_gen_synthetic_trace(E, k, B, S, skew, persistence, active_fraction, seed,
                                           _ptr(experts), _ptr(weights))
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return experts.reshape(B, S, k), weights.reshape(B, S, k)


def ref_save_synthetic_trace(path, E, k, B, S, skew, persistence, active_fraction, seed):
    rc = ref_lib().ref_save_synthetic_trace(E, k, B, S, skew, persistence, active_fraction, seed,
                                            str(path).encode())
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())


def ref_trace_roundtrip(in_path, out_path=""):
    """(E, k, batches) of a trace file loaded by the reference; re-saved to
    out_path when given.  Raises ValueError (invalid_argument) or OracleError."""
    dims = np.zeros(3, np.int32)
    rc = ref_lib().ref_trace_roundtrip(str(in_path).encode(), str(out_path).encode(), _ptr(dims))
    if rc == 1:
        raise ValueError(ref_lib().ref_last_error().decode())
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return tuple(int(v) for v in dims)


def ref_trace_loads(path, E, B):
    share = np.zeros(E * B, np.float64)
    rc = ref_lib().ref_trace_loads(str(path).encode(), _ptr(share), E * B)
    if rc:
        raise OracleError(ref_lib().ref_last_error().decode())
    return share.reshape(B, E).T


# --------------------------------------------------------------- C restatement
def c_dynamic_dispatch(experts: np.ndarray, E: int):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    order = np.zeros(max(S * k, 1), np.int32)
    counts = np.zeros(max(E, 1), np.int32)
    splits = np.zeros(max(E + 1, 1), np.int32)
    pos = np.zeros(max(S * k, 1), np.int32)
    rc = c_oracle().or_dynamic_dispatch(_ptr(ex), S, k, E, _ptr(order), _ptr(counts), _ptr(splits),
                                        _ptr(pos))
    if rc:
        raise OracleError(c_oracle().or_last_error().decode())
    return order[:S * k], counts[:E], splits[:E + 1], pos[:S * k]


def c_static_dispatch(experts: np.ndarray, E: int, C_: float):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    cap0 = c_oracle().or_expert_capacity(C_, S) if C_ > 0 else 1
    slots = np.zeros(max(E * max(cap0, 1), 1), np.int32)
    dropped = np.zeros(2 * S * k + 2, np.int32)
    pos = np.zeros(max(S * k, 1), np.int32)
    cap = C.c_int(0)
    nd = C.c_int(0)
    rc = c_oracle().or_static_dispatch(_ptr(ex), S, k, E, C_, C.byref(cap), _ptr(slots), slots.size,
                                       _ptr(dropped), C.byref(nd), _ptr(pos))
    if rc:
        raise OracleError(c_oracle().or_last_error().decode())
    c = cap.value
    return c, slots[:E * c].reshape(E, c), dropped[:2 * nd.value].reshape(-1, 2), pos[:S * k]


def c_exchange_counts(experts, D, device_of):
    ex = np.ascontiguousarray(experts, dtype=np.int32)
    S, k = ex.shape
    dev = np.ascontiguousarray(device_of, dtype=np.int32)
    out = np.zeros(D * D, np.int64)
    c_oracle().or_exchange_counts(_ptr(ex), S, k, D, _ptr(dev), _ptr(out))
    return out.reshape(D, D)
