"""Oracle attention over a token-slot KV pool (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

What the hot path computes has a plain definition: exact causal softmax
attention ("KV cache computation depends only on prefix
tokens"; prefill / decode).  The paged pool and prefix reuse must reach exactly
this result faster.  Written out per query row, per q head, in float64:

    g     = h // (H_q / H_kv)                               (R14: contiguous GQA groups)
    s_j   = scale * sum_d q[d] * K[rtt[r, j], g, d]          j = 0..p   (R13: causal)
    w_j   = exp(s_j - max s) / sum_j exp(s_j - max s)
    o     = sum_j w_j * V[rtt[r, j], g, :]

Extend first writes k_new / v_new into the pool at rtt[r, prefix_len + j]
(one token per page), then attends.  Decode attends for the one
query at p = seq_len - 1 (its KV already stored).

Each (row, kv-group) evaluation uses fixed array shapes that depend only on p,
so the same query computed with or without prefix reuse runs the identical
sequence of floating-point operations: reuse invariance is bitwise.
"""
from __future__ import annotations

import numpy as np


class OraclePool:
    """The oracle's own KV pool: K and V as float32 [S, H_kv, hd] (holds bf16 values exactly)."""

    def __init__(self, num_slots: int, h_kv: int, head_dim: int):
        self.k = np.zeros((num_slots, h_kv, head_dim), dtype=np.float32)
        self.v = np.zeros((num_slots, h_kv, head_dim), dtype=np.float32)

    def store(self, slots, k_new, v_new):
        """k_pool[slot] = k_new; v_pool[slot] = v_new (one token per page)."""
        slots = np.asarray(slots, dtype=np.int64)
        self.k[slots] = np.asarray(k_new, dtype=np.float32)
        self.v[slots] = np.asarray(v_new, dtype=np.float32)


def attend_row(q_group: np.ndarray, kmat: np.ndarray, vmat: np.ndarray, scale: float) -> np.ndarray:
    """Softmax attention of G query heads (float64 [G, hd]) over keys/values [n, hd]."""
    s = (q_group @ kmat.T) * scale                  # [G, n]
    m = s.max(axis=1, keepdims=True)
    e = np.exp(s - m)
    w = e / e.sum(axis=1, keepdims=True)
    return w @ vmat                                  # [G, hd]


def extend(pool: OraclePool, rtt_rows, prefix_lens, extend_lens, q, k_new, v_new, h_q: int, h_kv: int,
           scale: float) -> np.ndarray:
    """Extend attention for a ragged batch.

    rtt_rows[r]  : int array of slots for positions 0..prefix_len+extend_len-1 of request r
    q            : [sum extend_lens, H_q, hd]  (ragged-packed in request order)
    k_new, v_new : [sum extend_lens, H_kv, hd]
    Returns o as float64 [sum extend_lens, H_q, hd].
    """
    q = np.asarray(q, dtype=np.float64)
    k_new = np.asarray(k_new)
    v_new = np.asarray(v_new)
    G = h_q // h_kv
    hd = q.shape[2]
    out = np.zeros((q.shape[0], h_q, hd), dtype=np.float64)
    off = 0
    for r, (pre, n) in enumerate(zip(prefix_lens, extend_lens)):
        row = np.asarray(rtt_rows[r], dtype=np.int64)
        pool.store(row[pre:pre + n], k_new[off:off + n], v_new[off:off + n])
        for j in range(n):
            p = pre + j
            slots = row[:p + 1]
            for g in range(h_kv):
                kmat = pool.k[slots, g].astype(np.float64)
                vmat = pool.v[slots, g].astype(np.float64)
                out[off + j, g * G:(g + 1) * G] = attend_row(q[off + j, g * G:(g + 1) * G], kmat, vmat, scale)
        off += n
    return out


def decode(pool: OraclePool, rtt_rows, seq_lens, q, h_q: int, h_kv: int, scale: float) -> np.ndarray:
    """Decode attention: one query per request at p = seq_len - 1.  q: [B, H_q, hd] -> float64 [B, H_q, hd]."""
    q = np.asarray(q, dtype=np.float64)
    G = h_q // h_kv
    out = np.zeros(q.shape, dtype=np.float64)
    for b, L in enumerate(seq_lens):
        if L < 1:
            raise ValueError("seq_len must be >= 1")
        slots = np.asarray(rtt_rows[b], dtype=np.int64)[:L]
        for g in range(h_kv):
            kmat = pool.k[slots, g].astype(np.float64)
            vmat = pool.v[slots, g].astype(np.float64)
            out[b, g * G:(g + 1) * G] = attend_row(q[b, g * G:(g + 1) * G], kmat, vmat, scale)
    return out
