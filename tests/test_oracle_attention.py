"""Pins for the oracle attention (oracle/attention.py, oracle/driver.py).

1. brute force without reuse: regenerate each request's full token list, build
   contiguous K/V straight from the generator (no pool, no tree, no slots) and
   run a differently written textbook softmax(Q K^T * scale) V with an explicit
   causal mask over the whole sequence;
2. reuse invariance: the same rows computed with prefix reuse and with full
   recompute are BITWISE equal;
3. a library special case: torch scaled_dot_product_attention in float64;
4. exact special cases: seq_len 1 => o = v_0; q = 0 => o = mean(V); identical
   keys => mean(V); one dominant key => its value; decode == extend(prefix=L-1, n=1).
"""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from oracle.driver import OracleEngine
from rxgen import workloads
from rxgen.hashing import prefix_hashes
from rxgen.values import gen_values, KIND_K, KIND_V, KIND_Q


def _brute(tokens, seed, shape, q_scale=1.0):
    """Full causal attention over the whole token list, no pool: [n, H_q, hd] float64."""
    h = prefix_hashes(tokens, seed)
    hd = shape.head_dim
    K = gen_values(h, range(shape.h_kv), KIND_K, hd).double().numpy()
    V = gen_values(h, range(shape.h_kv), KIND_V, hd).double().numpy()
    Q = gen_values(h, range(shape.h_q), KIND_Q, hd, scale=q_scale).double().numpy()
    n = len(tokens)
    out = np.zeros((n, shape.h_q, hd))
    mask = np.tril(np.ones((n, n), dtype=bool))
    for hq in range(shape.h_q):
        g = hq * shape.h_kv // shape.h_q
        S = Q[:, hq, :] @ K[:, g, :].T * shape.sm_scale
        S = np.where(mask, S, -np.inf)
        S = S - S.max(axis=1, keepdims=True)
        P = np.exp(S)
        P /= P.sum(axis=1, keepdims=True)
        out[:, hq, :] = P @ V[:, g, :]
    return out


def _all_rows(call, seqs):
    return [(i, j) for i, s in enumerate(seqs) for j in range(s.n_prompt - s.prefix_len)]


def _all_dec(call, step, running):
    return list(range(len(running)))


@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_engine_vs_brute_force_c1_small(q_scale):
    wl = workloads.c1(seed=1, n_req=4, prefix=12, new=5, decode=3, num_slots=256)
    eng = OracleEngine(wl, sample_extend=_all_rows, sample_decode=_all_dec, q_scale=q_scale)
    eng.run_workload()
    reqs = wl.phases[1][1]
    # final token lists of the batch requests: prompt + 3 generated tokens
    # (recover them from the engine's finished trace by re-running the mock model)
    from oracle.driver import Seq
    for bi, r in enumerate(reqs):
        s = Seq(0, r.prompt, r.max_new_tokens, wl.seed, wl.vocab)
        for _ in range(r.max_new_tokens):
            s.gen_next()
        full = _brute(s.tokens, wl.seed, wl.shape, q_scale)
        # batch extend is the 2nd extend call; prefix 12 cached -> rows 12..16
        for j in range(5):
            got = eng.outputs[("extend", 1, bi, j)]
            np.testing.assert_allclose(got, full[12 + j], rtol=0, atol=1e-12)
        for t in range(3):
            got = eng.outputs[("decode", t, bi)]
            np.testing.assert_allclose(got, full[17 + t], rtol=0, atol=1e-12)
    # the hint extend covered rows 0..11 of the shared prefix
    for j in range(12):
        full = _brute(list(wl.phases[0][1][0].prompt), wl.seed, wl.shape, q_scale)
        np.testing.assert_allclose(eng.outputs[("extend", 0, 0, j)], full[j], rtol=0, atol=1e-12)


def test_reuse_invariance_bitwise():
    rng = np.random.default_rng(3)
    h_q, h_kv, hd = 4, 2, 32
    n_pre, n_new, S = 9, 6, 64
    toks = rng.integers(1, 1000, n_pre + n_new)
    h = prefix_hashes(toks, 11)
    K = gen_values(h, range(h_kv), KIND_K, hd).float().numpy()
    V = gen_values(h, range(h_kv), KIND_V, hd).float().numpy()
    Q = gen_values(h, range(h_q), KIND_Q, hd).float().numpy()
    scale = 1 / math.sqrt(hd)
    row = rng.permutation(np.arange(1, S))[:n_pre + n_new]
    # full recompute (prefix 0)
    p1 = A.OraclePool(S, h_kv, hd)
    o_full = A.extend(p1, [row], [0], [n_pre + n_new], Q, K, V, h_q, h_kv, scale)
    # reuse: prefix KV already in the pool, extend only the new tokens
    p2 = A.OraclePool(S, h_kv, hd)
    p2.store(row[:n_pre], K[:n_pre], V[:n_pre])
    o_reuse = A.extend(p2, [row], [n_pre], [n_new], Q[n_pre:], K[n_pre:], V[n_pre:], h_q, h_kv, scale)
    assert np.array_equal(o_full[n_pre:], o_reuse)
    # decode of the last position equals extend's last row, bitwise
    o_dec = A.decode(p2, [row], [n_pre + n_new], Q[-1:], h_q, h_kv, scale)
    assert np.array_equal(o_dec[0], o_reuse[-1])


def test_sdpa_float64_special_case():
    rng = np.random.default_rng(4)
    h_q, h_kv, hd, L = 8, 2, 64, 40
    K = rng.standard_normal((L, h_kv, hd)).astype(np.float32)
    V = rng.standard_normal((L, h_kv, hd)).astype(np.float32)
    Q = rng.standard_normal((L, h_q, hd)).astype(np.float32)
    row = np.arange(1, L + 1)
    pool = A.OraclePool(L + 1, h_kv, hd)
    o = A.extend(pool, [row], [0], [L], Q, K, V, h_q, h_kv, 0.125)
    q = torch.from_numpy(Q).double().transpose(0, 1)                 # [H_q, L, hd]
    k = torch.from_numpy(K).double().transpose(0, 1).repeat_interleave(h_q // h_kv, 0)
    v = torch.from_numpy(V).double().transpose(0, 1).repeat_interleave(h_q // h_kv, 0)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=0.125)
    np.testing.assert_allclose(o, ref.transpose(0, 1).numpy(), rtol=0, atol=1e-12)


def test_exact_special_cases():
    rng = np.random.default_rng(5)
    h_q, h_kv, hd = 4, 1, 16
    K = rng.standard_normal((6, h_kv, hd)).astype(np.float32)
    V = rng.standard_normal((6, h_kv, hd)).astype(np.float32)
    pool = A.OraclePool(8, h_kv, hd)
    pool.store(np.arange(1, 7), K, V)
    row = [np.arange(1, 7)]
    q = rng.standard_normal((1, h_q, hd))
    # seq_len 1: the single weight is exactly 1
    o = A.decode(pool, row, [1], q, h_q, h_kv, 0.25)
    assert np.array_equal(o[0], np.repeat(V[0:1, 0].astype(np.float64), h_q, 0))
    # q = 0: uniform weights -> mean of V
    o = A.decode(pool, row, [6], np.zeros((1, h_q, hd)), h_q, h_kv, 0.25)
    np.testing.assert_allclose(o[0], np.repeat(V[:, 0].astype(np.float64).mean(0, keepdims=True), h_q, 0), atol=1e-14)
    # identical keys -> mean of V regardless of q
    pool.store(np.arange(1, 7), np.repeat(K[:1], 6, 0), V)
    o = A.decode(pool, row, [6], q, h_q, h_kv, 0.25)
    np.testing.assert_allclose(o[0], np.repeat(V[:, 0].astype(np.float64).mean(0, keepdims=True), h_q, 0), atol=1e-14)
    # one dominant key -> its value
    K2 = np.zeros((6, h_kv, hd), np.float32)
    K2[3, 0, 0] = 1000.0
    pool.store(np.arange(1, 7), K2, V)
    qd = np.zeros((1, h_q, hd))
    qd[0, :, 0] = 1.0
    o = A.decode(pool, row, [6], qd, h_q, h_kv, 1.0)
    np.testing.assert_allclose(o[0], np.repeat(V[3:4, 0], h_q, 0), atol=1e-12)
