"""numpy restatement of the MoE-layer arithmetic -- TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED by the reference: the reference simulator has no gate, softmax,
top-k, expert FFN or weighted sum ("actual neural network execution
... out of scope").  This module follows the paper:

* gate + top-k: PAPER.md:178-187 ("a gating function decides which expert(s)
  ... top-1 or top-2"); the routing it produces must satisfy the reference's
  TokenAssignment invariants (proj/src/trace.cpp:47-67: k distinct ids in
  [0,E), weights >= 0 summing to 1 within 1e-9).
  Decisions (documented in DESIGN.md): ties -> lower expert id; slot j orders
  the selected experts by descending logit; weights are the softmax restricted
  to the k selected logits (the full-softmax normaliser cancels); the last
  weight is 1 - sum(others).
* dispatch: the reference's own dynamic_dispatch (gating.cpp:58-86; callers
  pass oracle.native.ref_dynamic_dispatch or the C restatement).
* expert FFN: H = relu(x W1_e^T), y = H W2_e^T ("FFN block";
  activation unspecified by the paper -> ReLU, no bias).
* combine: out[t] = sum_j w[t,j] * y[t,j] in slot order j (gating.hpp:107-141
  restores slot order; the weighted sum is the paper's combine).

Synthetic data (``synth``) is a counter-based generator bit-identical to the
CUDA fill kernel (paper_2303_06182_b200/csrc/rowops.cu), so CPU and GPU see the
same bf16 inputs without shipping them.
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15
TID = 0xD1B54A32D192ED03

# tensor ids for synth()
T_X, T_WG, T_W1, T_W2 = 1, 2, 3, 4


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def synth_f32(n_or_index, seed: int, tensor_id: int, scale: float) -> np.ndarray:
    """fp32 values (before bf16 rounding) for element indices ``idx``.

    value(i) = (int(h >> 40) - 2^23) * 2^-23 * scale with
    h = mix64(seed*PHI + tensor_id*TID + i)  (all mod 2^64).
    """
    if np.isscalar(n_or_index):
        idx = np.arange(int(n_or_index), dtype=np.uint64)
    else:
        idx = np.asarray(n_or_index, dtype=np.uint64)
    base = np.uint64(((seed * PHI) + (tensor_id * TID)) & M64)
    with np.errstate(over="ignore"):
        h = _mix64(idx + base)
    u = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    x = u.astype(np.float32) * np.float32(2.0 ** -23)
    return (x * np.float32(scale)).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (round-to-nearest-even), returned as uint16 bits."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((b >> np.uint32(16)) & np.uint32(1)) + np.uint32(0x7FFF)
    with np.errstate(over="ignore"):
        out = ((b + rounding) >> np.uint32(16)).astype(np.uint16)
    nan = np.isnan(np.ascontiguousarray(x, dtype=np.float32))
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (np.asarray(u16, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def synth_bf16(shape, seed: int, tensor_id: int, scale: float, index_offset: int = 0) -> np.ndarray:
    """bf16 bits (uint16) with the given shape; element i of the flattened
    tensor uses counter index_offset + i."""
    n = int(np.prod(shape))
    idx = np.arange(index_offset, index_offset + n, dtype=np.uint64)
    return bf16_round(synth_f32(idx, seed, tensor_id, scale)).reshape(shape)


def init_scales(TD: int, HD: int):
    """Uniform half-widths giving std 1 (X), 1/sqrt(TD) (Wg), sqrt(2/TD) (W1),
    1/sqrt(HD) (W2): a = sqrt(3) * std."""
    r3 = math.sqrt(3.0)
    return {"x": r3, "wg": r3 / math.sqrt(TD), "w1": r3 * math.sqrt(2.0 / TD), "w2": r3 / math.sqrt(HD)}


# ------------------------------------------------------------------ gate
def topk_from_logits(logits: np.ndarray, k: int):
    """k largest per row, ties -> lower id, slot j by descending logit.
    Returns (idx int32 [S,k], w float64 [S,k])."""
    L = np.asarray(logits, dtype=np.float32)
    S, E = L.shape
    # stable sort on -logit keeps lower ids first among equal logits
    order = np.argsort(-L, axis=1, kind="stable")[:, :k].astype(np.int32)
    sel = np.take_along_axis(L, order, axis=1).astype(np.float64)
    ex = np.exp(sel - sel[:, :1])
    w = ex / ex.sum(axis=1, keepdims=True)
    if k > 1:
        w[:, -1] = 1.0 - w[:, :-1].sum(axis=1)
    else:
        w[:, 0] = 1.0
    return order, w


def gate_logits(X: np.ndarray, Wg: np.ndarray) -> np.ndarray:
    """fp32 logits = X Wg^T (X, Wg already as fp32 values)."""
    return (X.astype(np.float32) @ Wg.astype(np.float32).T).astype(np.float32)


# ------------------------------------------------------------------ FFN
def expert_ffn(x: np.ndarray, w1: np.ndarray, w2: np.ndarray, round_h_bf16: bool = False) -> np.ndarray:
    """y = relu(x w1^T) w2^T in fp32 (x [n,TD], w1 [HD,TD], w2 [TD,HD])."""
    h = np.maximum(x.astype(np.float32) @ w1.astype(np.float32).T, 0.0).astype(np.float32)
    if round_h_bf16:
        h = bf16_to_f32(bf16_round(h))
    return (h @ w2.astype(np.float32).T).astype(np.float32)


def layer_forward(X, W1, W2, idx, w, E, tokens=None, round_h_bf16=False):
    """fp32 MoE layer output for the given routing (idx [S,k], w [S,k]).

    X [S,TD], W1 [E,HD,TD], W2 [E,TD,HD] as fp32 arrays (or callables
    e -> (w1, w2) for lazily materialised experts).  ``tokens`` restricts the
    computation to a subset of token rows (returned in that order).
    """
    S, k = idx.shape
    toks = np.arange(S) if tokens is None else np.asarray(tokens)
    TD = X.shape[1]
    out = np.zeros((len(toks), TD), np.float32)
    # group the requested (token, j) pairs by expert, then one GEMM per expert
    pairs = {}
    for r, t in enumerate(toks):
        for j in range(k):
            pairs.setdefault(int(idx[t, j]), []).append((r, t, j))
    contrib = np.zeros((len(toks), k, TD), np.float32)
    for e, lst in pairs.items():
        if callable(W1):
            w1, w2 = W1(e), W2(e)
        else:
            w1, w2 = W1[e], W2[e]
        rows = np.array([t for (_, t, _) in lst])
        y = expert_ffn(X[rows], w1, w2, round_h_bf16)
        for n, (r, t, j) in enumerate(lst):
            contrib[r, j] = np.float32(w[t, j]) * y[n]
    for j in range(k):  # slot order, fp32 accumulate
        out += contrib[:, j]
    return out


def rel_fro(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
