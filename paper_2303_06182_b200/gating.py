"""Python host mirror of the reference's gating API (proj/include/moesim/
gating.hpp, trace.hpp), on top of the C ABI -- the GPU does the dispatch.

Same names, argument meaning and error behaviour as the reference, so the
parity tests read like ``proj/tests/test_gating.cpp``:

  GatingMode, GatingConfig         gating.hpp:16-23
  TokenAssignment, Batch           trace.hpp:15-25
  expert_capacity                  gating.hpp:31,   gating.cpp:22-28
  StaticDispatchPlan               gating.hpp:36-47 (slots is [E, cap], -1 = placeholder)
  DynamicDispatchPlan              gating.hpp:53-60
  static_dispatch/dynamic_dispatch gating.hpp:68-69, gating.cpp:30-86
  waste_factor                     gating.hpp:71,   gating.cpp:88-92
  dispatch_mask_elements           gating.hpp:74,   gating.cpp:94-99
  dispatch_cost_counts             gating.hpp:85,   gating.cpp:101-125
  debug_json                       gating.hpp:89-90, gating.cpp:127-153
  combine                          gating.hpp:107-184

Errors: the reference's std::invalid_argument becomes ``InvalidArgument``
(a ValueError) carrying the reference's exact message text.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np

from ._capi import MoeInvalidArgument, check, load

kPlaceholder = -1


class InvalidArgument(ValueError):
    pass


class GatingMode(enum.Enum):
    kStatic = 0
    kDynamic = 1


@dataclass
class GatingConfig:
    num_experts: int = 0
    top_k: int = 1
    capacity_factor: float = 1.0
    mode: GatingMode = GatingMode.kDynamic


@dataclass
class TokenAssignment:
    experts: list
    weights: list


@dataclass
class Batch:
    tokens: list = field(default_factory=list)
    batch_id: int = 0

    def seq_len(self) -> int:
        return len(self.tokens)


@dataclass
class StaticDispatchPlan:
    seq_len: int = 0
    num_experts: int = 0
    top_k: int = 1
    capacity: int = 0
    slots: np.ndarray = None  # [E, cap] int32
    dropped: list = field(default_factory=list)

    def placed(self) -> int:
        return int((self.slots != kPlaceholder).sum())


@dataclass
class DynamicDispatchPlan:
    seq_len: int = 0
    num_experts: int = 0
    top_k: int = 1
    order: list = field(default_factory=list)
    counts: list = field(default_factory=list)
    splits: list = field(default_factory=list)


@dataclass
class WasteFactor:
    value: float = 0.0


@dataclass
class DispatchCostCounts:
    comparisons: int = 0
    count_passes: int = 0
    gather_elements: int = 0


@dataclass
class CombinedEntry:
    expert: int
    weight: float
    payload: Any


_ctx = None


def _context():
    global _ctx
    if _ctx is None:
        h = C.c_void_p()
        check(load().moe_ctx_create(0, C.byref(h)))
        _ctx = h
    return _ctx


def _call(status):
    try:
        check(status)
    except MoeInvalidArgument as e:
        raise InvalidArgument(e.msg) from None


def _check_batch(batch: Batch, cfg: GatingConfig):
    # gating.cpp:12-18 (message text verbatim)
    if cfg.num_experts < 1:
        raise InvalidArgument("num_experts must be positive")
    if cfg.top_k < 1:
        raise InvalidArgument("top_k must be positive")
    if cfg.top_k > cfg.num_experts:
        raise InvalidArgument("top_k exceeds num_experts")
    if not batch.tokens:
        raise InvalidArgument("empty batch")


def _flat_experts(batch: Batch, k: int) -> np.ndarray:
    ex = np.empty(len(batch.tokens) * k, np.int32)
    for t, ta in enumerate(batch.tokens):
        ex[t * k:(t + 1) * k] = ta.experts[:k]
    return ex


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def expert_capacity(capacity_factor: float, seq_len: int) -> int:
    return int(load().moe_expert_capacity(float(capacity_factor), int(seq_len)))


def dynamic_dispatch(batch: Batch, cfg: GatingConfig) -> DynamicDispatchPlan:
    _check_batch(batch, cfg)
    if cfg.mode != GatingMode.kDynamic:
        raise InvalidArgument("dynamic_dispatch requires dynamic mode")
    S, k, E = batch.seq_len(), cfg.top_k, cfg.num_experts
    ex = _flat_experts(batch, k)
    order = np.empty(S * k, np.int32)
    counts = np.empty(E, np.int32)
    splits = np.empty(E + 1, np.int32)
    _call(load().moe_dynamic_dispatch_host(_context(), _ptr(ex), S, k, E, _ptr(order),
                                           _ptr(counts), _ptr(splits)))
    return DynamicDispatchPlan(S, E, k, order.tolist(), counts.tolist(), splits.tolist())


def static_dispatch(batch: Batch, cfg: GatingConfig) -> StaticDispatchPlan:
    _check_batch(batch, cfg)
    if cfg.mode != GatingMode.kStatic:
        raise InvalidArgument("static_dispatch requires static mode")
    if cfg.capacity_factor <= 0.0:
        raise InvalidArgument("capacity factor must be positive in static mode")
    S, k, E = batch.seq_len(), cfg.top_k, cfg.num_experts
    cap = expert_capacity(cfg.capacity_factor, S)
    if cap <= 0:
        raise InvalidArgument("zero capacity")
    ex = _flat_experts(batch, k)
    slots = np.empty(E * cap, np.int32)
    dropped = np.empty(2 * S * k + 2, np.int32)
    capo = C.c_int32(0)
    nd = C.c_int32(0)
    _call(load().moe_static_dispatch_host(_context(), _ptr(ex), S, k, E, float(cfg.capacity_factor),
                                          C.byref(capo), _ptr(slots), slots.size, _ptr(dropped),
                                          C.byref(nd)))
    drops = [(int(dropped[2 * i]), int(dropped[2 * i + 1])) for i in range(nd.value)]
    return StaticDispatchPlan(S, E, k, cap, slots.reshape(E, cap), drops)


def waste_factor(num_experts: int, capacity_factor: float, top_k: int) -> WasteFactor:
    if num_experts <= 0 or capacity_factor <= 0.0 or top_k <= 0:
        raise InvalidArgument("waste_factor requires positive inputs")
    return WasteFactor(num_experts * capacity_factor / top_k)


def dispatch_mask_elements(seq_len: int, num_experts: int, capacity_factor: float) -> int:
    if seq_len <= 0 or num_experts <= 0 or capacity_factor <= 0.0:
        raise InvalidArgument("dispatch_mask_elements requires positive inputs")
    return num_experts * seq_len * expert_capacity(capacity_factor, seq_len)


def _inverse(order: Sequence[int], n_slots: int) -> np.ndarray:
    o = np.ascontiguousarray(np.asarray(order, dtype=np.int32).reshape(-1))
    pos = np.empty(max(n_slots, 1), np.int32)
    _call(load().moe_inverse_order_host(_context(), _ptr(o), o.size, _ptr(pos), n_slots))
    return pos[:n_slots]


def combine(plan, batch: Batch, outputs: Sequence[Any]):
    """gating.hpp:107-184: restore expert outputs to token order; every token
    receives its entries in assignment-slot order (the GPU computes the
    inverse permutation; payloads are opaque, as in the reference)."""
    k = plan.top_k
    if isinstance(plan, DynamicDispatchPlan):
        total = plan.seq_len * k
        if len(outputs) != total:
            raise InvalidArgument("combine: payload count mismatch vs. plan")
        if batch.seq_len() != plan.seq_len:
            raise InvalidArgument("combine: batch does not match plan")
        pos = _inverse(plan.order, total)
    else:
        total = plan.num_experts * plan.capacity
        if len(outputs) != total:
            raise InvalidArgument("combine: payload count mismatch vs. plan")
        if batch.seq_len() != plan.seq_len:
            raise InvalidArgument("combine: batch does not match plan")
        pos = _inverse(plan.slots.reshape(-1), plan.seq_len * k)
    result = []
    for t, ta in enumerate(batch.tokens):
        entries = []
        for j in range(k):
            p = int(pos[t * k + j])
            if p >= 0:
                e = ta.experts[j] if isinstance(plan, DynamicDispatchPlan) else p // plan.capacity
                entries.append(CombinedEntry(e, ta.weights[j], outputs[p]))
        result.append(entries)
    return result


def dispatch_cost_counts(plan: DynamicDispatchPlan, token_dim: int) -> DispatchCostCounts:
    """gating.cpp:101-125 instrumentation.  ``comparisons`` is measured by
    re-running std::stable_sort over the plan's expert keys, exactly as the
    reference does -- inside the C++ drop-in library (libmoesim_b200.so)."""
    if token_dim <= 0:
        raise InvalidArgument("token_dim must be positive")
    total = plan.seq_len * plan.top_k
    key = np.zeros(max(total, 1), np.int32)
    for e in range(plan.num_experts):
        for p in range(plan.splits[e], plan.splits[e + 1]):
            key[plan.order[p]] = e
    comps = int(_cxx().moesim_stable_sort_comparisons(_ptr(key), total))
    return DispatchCostCounts(comps, total, total * token_dim)


_CXX = None


def _cxx():
    global _CXX
    if _CXX is None:
        import os

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmoesim_b200.so")
        load()
        _CXX = C.CDLL(path)
        _CXX.moesim_stable_sort_comparisons.restype = C.c_int64
        _CXX.moesim_stable_sort_comparisons.argtypes = [C.c_void_p, C.c_int]
    return _CXX


def debug_json(plan) -> str:
    """gating.cpp:127-153: one line, keys sorted (nlohmann's std::map order)."""
    if isinstance(plan, DynamicDispatchPlan):
        d = {"counts": list(plan.counts), "num_experts": plan.num_experts, "order": list(plan.order),
             "seq_len": plan.seq_len, "splits": list(plan.splits), "top_k": plan.top_k}
    else:
        d = {"capacity": plan.capacity, "dropped": [[t, e] for (t, e) in plan.dropped],
             "num_experts": plan.num_experts, "seq_len": plan.seq_len,
             "slots": plan.slots.tolist(), "top_k": plan.top_k}
    return json.dumps(d, separators=(",", ":"), sort_keys=True)
