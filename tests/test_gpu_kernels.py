"""GPU parity: librx kernels (through the C ABI) against the fp64 oracle.

Tolerance (BASELINE.json north star): max-abs 2e-2 and mean-abs 2e-3 on the
bf16 outputs vs the oracle's fp64 result; plus relative-error and peaked
(q x 4) variants (reading R19).  Stores are checked bit-exact.  Inputs are
rxgen values (seeded, synthetic); slots are deliberately fragmented or
contiguous to hit both gather paths of the extend kernel, and lengths are
ragged (tile tails, splits).
"""
import math

import numpy as np
import pytest
import torch

from oracle import attention as A
from rxgen.values import gen_values, KIND_K, KIND_V, KIND_Q

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2312_07104_b200 as rx

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _vals(rng, n, heads, kind, hd, scale=1.0):
    h = rng.integers(0, 2**63, n, dtype=np.uint64)
    return gen_values(h, range(heads), kind, hd, scale=scale)


def _cmp(got_bf16, ref64, tag=""):
    got = got_bf16.float().cpu().double().numpy()
    err = np.abs(got - ref64)
    assert np.isfinite(got).all(), tag
    assert err.max() <= MAX_ABS, f"{tag} max-abs {err.max()}"
    assert err.mean() <= MEAN_ABS, f"{tag} mean-abs {err.mean()}"
    return err.max(), err.mean()


def _pool(S, h_kv, hd, rng):
    k = torch.zeros((S, h_kv, hd), dtype=torch.bfloat16)
    v = torch.zeros_like(k)
    return k, v


def test_store_kv_bit_exact():
    rng = np.random.default_rng(0)
    S, h_kv, hd, n = 500, 4, 128, 77
    cfg = rx.attn_cfg(8, h_kv, hd, 1 / math.sqrt(hd))
    kp = torch.zeros((S, h_kv, hd), dtype=torch.bfloat16, device="cuda")
    vp = torch.zeros_like(kp)
    slots = rng.permutation(np.arange(1, S))[:n].astype(np.int32)
    k = _vals(rng, n, h_kv, KIND_K, hd).cuda()
    v = _vals(rng, n, h_kv, KIND_V, hd).cuda()
    rtt = torch.zeros((4, 64), dtype=torch.int32, device="cuda")
    idx = torch.from_numpy(rng.permutation(256)[:n].astype(np.int64)).cuda()
    rx.rx_store_kv(cfg, torch.from_numpy(slots).cuda(), k, v, kp, vp, rtt, idx)
    torch.cuda.synchronize()
    assert torch.equal(kp[torch.from_numpy(slots).long().cuda()], k)
    assert torch.equal(vp[torch.from_numpy(slots).long().cuda()], v)
    assert torch.equal(rtt.view(-1)[idx], torch.from_numpy(slots).cuda())
    untouched = np.setdiff1d(np.arange(S), slots)
    assert kp[torch.from_numpy(untouched).cuda()].abs().sum().item() == 0


def test_copy_h2d_bitwise():
    """rx_copy_h2d (SM-driven upload of pinned host metadata): every byte arrives, for aligned and
    unaligned sizes / offsets; pageable host memory is refused."""
    rng = np.random.default_rng(2)
    for n in (1, 15, 16, 4097, 3 << 20):
        h = torch.from_numpy(rng.integers(0, 256, n + 3, dtype=np.uint8)).pin_memory()
        for off in (0, 3):
            src = h[off:off + n]
            d = torch.empty(n, dtype=torch.uint8, device="cuda")
            rx.rx_copy_h2d(d, src)
            torch.cuda.synchronize()
            assert torch.equal(d.cpu(), src)
    with pytest.raises(ValueError):
        rx.rx_copy_h2d(torch.empty(8, dtype=torch.uint8, device="cuda"), torch.zeros(8, dtype=torch.uint8))


def test_store_kv_table_only():
    """rx_store_kv with null k / v and a table index (the engine's jump-forward output steps, whose
    K/V the following rx_extend stores): only the table entries are written, the pools are not."""
    rng = np.random.default_rng(1)
    n = 50
    cfg = rx.attn_cfg(8, 4, 128, 1 / math.sqrt(128))
    slots = torch.from_numpy(rng.permutation(np.arange(1, 400))[:n].astype(np.int32)).cuda()
    rtt = torch.zeros((4, 64), dtype=torch.int32, device="cuda")
    idx = torch.from_numpy(rng.permutation(256)[:n].astype(np.int64)).cuda()
    rx.rx_store_kv(cfg, slots, None, None, None, None, rtt, idx)
    torch.cuda.synchronize()
    assert rx.rx_last_launch_count() == 1
    assert torch.equal(rtt.view(-1)[idx], slots)
    assert int((rtt != 0).sum()) == n


DEC_CASES = [
    # (h_q, h_kv, hd, seq_lens)
    (8, 2, 64, [1, 2, 15, 16, 17, 97, 300]),
    (32, 32, 128, [1, 5, 64, 129, 1600]),
    (32, 8, 128, [33, 511, 512, 513, 2000, 4100]),
    (64, 8, 128, [1, 17, 1000, 8300]),
    (16, 8, 128, [40, 700]),
    (8, 8, 64, [3, 1025]),
]


@pytest.mark.parametrize("h_q,h_kv,hd,lens", DEC_CASES)
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_decode_vs_oracle(h_q, h_kv, hd, lens, q_scale):
    rng = np.random.default_rng(len(lens) * 7 + hd + h_q)
    B = len(lens)
    S = sum(lens) + 64
    kall = _vals(rng, S, h_kv, KIND_K, hd)
    vall = _vals(rng, S, h_kv, KIND_V, hd)
    kall[0] = 0
    vall[0] = 0
    stride = max(lens) + 8
    rtt = np.zeros((B, stride), dtype=np.int32)
    perm = rng.permutation(np.arange(1, S))
    off = 0
    for b, L in enumerate(lens):
        rtt[b, :L] = perm[off:off + L]     # fragmented slots
        off += L
    q = _vals(rng, B, h_q, KIND_Q, hd, scale=q_scale)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    kp, vp = kall.cuda(), vall.cuda()
    o = torch.empty((B, h_q, hd), dtype=torch.bfloat16, device="cuda")
    ws_n = rx.rx_decode_workspace_bytes(cfg, B, max(lens))
    ws = torch.zeros(max(ws_n, 1), dtype=torch.uint8, device="cuda")
    rx.rx_decode(cfg, torch.from_numpy(rtt).cuda(), None, torch.tensor(lens, dtype=torch.int32, device="cuda"),
                 max(lens), q.cuda(), kp, vp, o, ws)
    torch.cuda.synchronize()
    pool = A.OraclePool(S, h_kv, hd)
    pool.store(np.arange(S), kall.float().numpy(), vall.float().numpy())
    ref = A.decode(pool, [rtt[b] for b in range(B)], lens, q.float().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
    _cmp(o, ref, f"decode {h_q}/{h_kv}/{hd} {lens}")
    # exact special case: seq_len 1 -> o == v_0 bit for bit
    for b, L in enumerate(lens):
        if L == 1:
            G = h_q // h_kv
            exp = vall[rtt[b, 0]].repeat_interleave(G, 0)
            assert torch.equal(o[b].cpu(), exp)


def test_decode_rows_indirection():
    """d_rows selects table rows: permuting rows and seq_lens together permutes outputs."""
    rng = np.random.default_rng(11)
    h_q, h_kv, hd = 32, 8, 128
    lens = [100, 257, 31]
    S = 1000
    kp = _vals(rng, S, h_kv, KIND_K, hd).cuda()
    vp = _vals(rng, S, h_kv, KIND_V, hd).cuda()
    rtt = torch.from_numpy(rng.integers(1, S, (3, 300)).astype(np.int32)).cuda()
    q = _vals(rng, 3, h_q, KIND_Q, hd).cuda()
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    o1 = torch.empty((3, h_q, hd), dtype=torch.bfloat16, device="cuda")
    o2 = torch.empty_like(o1)
    ws = torch.zeros(rx.rx_decode_workspace_bytes(cfg, 3, 300) + 1, dtype=torch.uint8, device="cuda")
    rx.rx_decode(cfg, rtt, None, torch.tensor(lens, dtype=torch.int32, device="cuda"), 257, q, kp, vp, o1, ws)
    perm = [2, 0, 1]
    rx.rx_decode(cfg, rtt, torch.tensor(perm, dtype=torch.int32, device="cuda"),
                 torch.tensor([lens[i] for i in perm], dtype=torch.int32, device="cuda"), 257, q[perm].contiguous(),
                 kp, vp, o2, ws)
    torch.cuda.synchronize()
    assert torch.equal(o2, o1[perm])


EXT_CASES = [
    # (h_q, h_kv, hd, prefix_lens, extend_lens, contiguous_prefix)
    (8, 2, 64, [64] * 4, [32] * 4, True),
    (8, 2, 64, [0, 1, 63, 200], [1, 5, 33, 130], False),
    (32, 32, 128, [0, 128, 129], [128, 1, 200], True),
    (32, 32, 128, [300, 17], [129, 64], False),
    (32, 8, 128, [0, 256, 511], [300, 17, 130], False),
    (32, 8, 128, [384, 384], [100, 256], True),
    (64, 8, 128, [1000, 0], [40, 150], True),
    (64, 8, 128, [257, 513], [16, 17], False),
    (16, 8, 128, [10, 140], [140, 10], False),
]


def _short_segments(seed, B, max_ext, max_pre):
    r = np.random.default_rng(seed)
    pre = [int(x) for x in r.integers(0, max_pre + 1, B)]
    ext = [int(x) for x in r.integers(0, max_ext + 1, B)]
    pre[0], ext[0], ext[1] = 0, max_ext, 0          # no prefix; the widest segment; an empty one
    return pre, ext


# short segments with enough (request, kv head) pairs: rx_extend takes the multi-query decode
# kernel (max_ext * G <= 32, batch * h_kv >= 148): jump-forward edges of constrained decoding
EXT_CASES += [
    (32, 32, 128, *_short_segments(1, 8, 20, 700), False),     # G=1: up to 3 column tiles
    (32, 32, 128, *_short_segments(2, 6, 32, 300), True),      # 4 tiles
    (32, 8, 128, *_short_segments(3, 20, 8, 900), False),      # G=4
    (64, 8, 128, *_short_segments(4, 20, 4, 500), False),      # G=8
    (8, 2, 64, *_short_segments(5, 80, 8, 200), False),        # hd 64
]


@pytest.mark.parametrize("h_q,h_kv,hd,pre,ext,contig", EXT_CASES)
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_extend_vs_oracle(h_q, h_kv, hd, pre, ext, contig, q_scale):
    rng = np.random.default_rng(sum(pre) + sum(ext) + hd)
    B = len(pre)
    S = sum(pre) + sum(ext) + 300
    stride = max(p + e for p, e in zip(pre, ext)) + 3
    rtt = np.zeros((B, stride), dtype=np.int32)
    free = list(range(1, S)) if contig else list(rng.permutation(np.arange(1, S)))
    off = 0
    for b in range(B):
        n = pre[b] + ext[b]
        rtt[b, :n] = free[off:off + n]
        off += n
    kpool = _vals(rng, S, h_kv, KIND_K, hd)
    vpool = _vals(rng, S, h_kv, KIND_V, hd)
    N = sum(ext)
    q = _vals(rng, N, h_q, KIND_Q, hd, scale=q_scale)
    kn = _vals(rng, N, h_kv, KIND_K, hd)
    vn = _vals(rng, N, h_kv, KIND_V, hd)
    indptr = np.concatenate([[0], np.cumsum(ext)]).astype(np.int32)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    kp, vp = kpool.cuda(), vpool.cuda()
    o = torch.full((N, h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    rx.rx_extend(cfg, torch.from_numpy(rtt).cuda(), None, torch.tensor(pre, dtype=torch.int32, device="cuda"),
                 torch.tensor(ext, dtype=torch.int32, device="cuda"), torch.from_numpy(indptr).cuda(), N, max(ext),
                 max(pre), q.cuda(), kn.cuda(), vn.cuda(), kp, vp, o)
    torch.cuda.synchronize()
    pool = A.OraclePool(S, h_kv, hd)
    pool.store(np.arange(S), kpool.float().numpy(), vpool.float().numpy())
    ref = A.extend(pool, [rtt[b] for b in range(B)], pre, ext, q.float().numpy(), kn.float().numpy(),
                   vn.float().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
    _cmp(o, ref, f"extend {h_q}/{h_kv}/{hd} pre={pre} ext={ext}")
    # fused store: new rows landed in their slots bit-exact, prefix rows untouched
    for b in range(B):
        s_new = torch.from_numpy(rtt[b, pre[b]:pre[b] + ext[b]].astype(np.int64)).cuda()
        assert torch.equal(kp[s_new], kn[indptr[b]:indptr[b + 1]].cuda())
        assert torch.equal(vp[s_new], vn[indptr[b]:indptr[b + 1]].cuda())
        s_pre = torch.from_numpy(rtt[b, :pre[b]].astype(np.int64)).cuda()
        assert torch.equal(kp[s_pre], kpool[rtt[b, :pre[b]].astype(np.int64)].cuda())


def test_extend_decode_consistency():
    """decode(seq_lens) == extend(prefix = seq_len - 1, n = 1) within tolerance of each other."""
    rng = np.random.default_rng(3)
    h_q, h_kv, hd = 32, 8, 128
    lens = [1, 130, 700]
    B = len(lens)
    S = 2000
    kpool = _vals(rng, S, h_kv, KIND_K, hd).cuda()
    vpool = _vals(rng, S, h_kv, KIND_V, hd).cuda()
    rtt = np.zeros((B, 800), dtype=np.int32)
    off = 1
    for b, L in enumerate(lens):
        rtt[b, :L] = np.arange(off, off + L)
        off += L
    rtt_d = torch.from_numpy(rtt).cuda()
    q = _vals(rng, B, h_q, KIND_Q, hd).cuda()
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    od = torch.empty((B, h_q, hd), dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(rx.rx_decode_workspace_bytes(cfg, B, 800) + 1, dtype=torch.uint8, device="cuda")
    rx.rx_decode(cfg, rtt_d, None, torch.tensor(lens, dtype=torch.int32, device="cuda"), 700, q, kpool, vpool, od, ws)
    last = torch.from_numpy(np.array([rtt[b, L - 1] for b, L in enumerate(lens)], dtype=np.int64)).cuda()
    oe = torch.empty_like(od)
    rx.rx_extend(cfg, rtt_d, None, torch.tensor([L - 1 for L in lens], dtype=torch.int32, device="cuda"),
                 torch.ones(B, dtype=torch.int32, device="cuda"), torch.arange(B + 1, dtype=torch.int32, device="cuda"),
                 B, 1, max(lens) - 1, q, kpool[last].contiguous(), vpool[last].contiguous(), kpool.clone(),
                 vpool.clone(), oe)
    torch.cuda.synchronize()
    assert (od.float() - oe.float()).abs().max().item() < 2e-2


def test_unsupported_and_invalid():
    cfg = rx.attn_cfg(12, 4, 128, 0.1)                  # G = 3
    o = torch.empty((1, 12, 128), dtype=torch.bfloat16, device="cuda")
    z = torch.zeros((4, 4, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rx.RxError) as e:
        rx.rx_decode(cfg, torch.zeros((1, 4), dtype=torch.int32, device="cuda"), None,
                     torch.ones(1, dtype=torch.int32, device="cuda"), 1, o, z, z, o)
    assert e.value.status == -5
    cfg = rx.attn_cfg(8, 2, 96, 0.1)
    with pytest.raises(rx.RxError):
        rx.rx_decode(cfg, torch.zeros((1, 4), dtype=torch.int32, device="cuda"), None,
                     torch.ones(1, dtype=torch.int32, device="cuda"), 1, o, z, z, o)
    with pytest.raises(ValueError):
        rx.rx_decode(rx.attn_cfg(8, 2, 64, 0.1), torch.zeros((1, 4), dtype=torch.int32), None,
                     torch.ones(1, dtype=torch.int32), 1, o, z, z, o)


@pytest.mark.parametrize("h_q,h_kv,hd", [(32, 8, 128), (64, 8, 128), (32, 32, 128), (8, 2, 64)])
def test_extend_many_items_ragged(h_q, h_kv, hd):
    """Many (q tile, head, request) items per persistent CTA, ragged lengths, mixed
    contiguous / fragmented prefixes; peaked softmax (q x 4) to exercise O rescaling."""
    rng = np.random.default_rng(h_q * 7 + hd)
    B = 24
    pre = [int(x) for x in rng.integers(0, 700, B)]
    pre[0], pre[1] = 0, 128
    ext = [int(x) for x in rng.integers(1, 300, B)]
    S = sum(pre) + sum(ext) + 64
    stride = max(p + e for p, e in zip(pre, ext))
    rtt = np.zeros((B, stride), dtype=np.int32)
    order = np.concatenate([np.arange(1, S // 2), rng.permutation(np.arange(S // 2, S))])
    off = 0
    for b in range(B):
        n = pre[b] + ext[b]
        rtt[b, :n] = order[off:off + n]
        off += n
    kpool = _vals(rng, S, h_kv, KIND_K, hd)
    vpool = _vals(rng, S, h_kv, KIND_V, hd)
    N = sum(ext)
    q = _vals(rng, N, h_q, KIND_Q, hd, scale=4.0)
    kn = _vals(rng, N, h_kv, KIND_K, hd)
    vn = _vals(rng, N, h_kv, KIND_V, hd)
    indptr = np.concatenate([[0], np.cumsum(ext)]).astype(np.int32)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    kp, vp = kpool.cuda(), vpool.cuda()
    o = torch.full((N, h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    rx.rx_extend(cfg, torch.from_numpy(rtt).cuda(), None, torch.tensor(pre, dtype=torch.int32, device="cuda"),
                 torch.tensor(ext, dtype=torch.int32, device="cuda"), torch.from_numpy(indptr).cuda(), N, max(ext),
                 max(pre), q.cuda(), kn.cuda(), vn.cuda(), kp, vp, o)
    torch.cuda.synchronize()
    pool = A.OraclePool(S, h_kv, hd)
    pool.store(np.arange(S), kpool.float().numpy(), vpool.float().numpy())
    ref = A.extend(pool, [rtt[b] for b in range(B)], pre, ext, q.float().numpy(), kn.float().numpy(),
                   vn.float().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
    _cmp(o, ref, f"extend-many {h_q}/{h_kv}/{hd}")


@pytest.mark.parametrize("h_q,h_kv,hd,lens", [(32, 8, 128, [1, 40, 700, 3000]), (8, 2, 64, [2, 300]),
                                              (64, 8, 128, [8300, 5])])
def test_decode_append_equals_store_then_decode(h_q, h_kv, hd, lens):
    _decode_append_check(h_q, h_kv, hd, lens)


@pytest.mark.parametrize("h_q,h_kv,hd,B,shared,contig", [
    (64, 8, 128, 128, 8192, True),     # C5 shape: 128 requests on one 8k context
    (64, 8, 128, 13, 1000, False),
    (32, 32, 128, 64, 1536, True),     # C2 shape (G = 1)
    (32, 8, 128, 40, 700, False),
    (8, 2, 64, 16, 64, True),          # C1 shape
])
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_cascade_decode_vs_oracle(h_q, h_kv, hd, B, shared, contig, q_scale):
    """rx_decode_cascade_append (shared prefix attended once on the tensor cores,
    suffixes by the decode kernel, LSE merge) against the fp64 oracle; the KV
    append (pool rows, req_to_token entries) is bit-identical to rx_decode_append."""
    _cascade_decode_check(h_q, h_kv, hd, B, shared, contig, q_scale, 300)


@pytest.mark.parametrize("h_q,h_kv,hd,B,shared,max_suffix", [
    (64, 8, 128, 24, 2048, 3000),      # several suffix splits per request, ragged last splits
    (32, 32, 128, 7, 512, 1200),       # few requests
    (8, 2, 64, 33, 128, 700),          # hd 64 (6-stage rings)
])
def test_cascade_decode_long_suffix_vs_oracle(h_q, h_kv, hd, B, shared, max_suffix):
    """Cascade step with long, ragged suffixes (several suffix splits per request, short last
    splits, few units) — vs the fp64 oracle."""
    _cascade_decode_check(h_q, h_kv, hd, B, shared, False, 1.0, max_suffix)


def _cascade_decode_check(h_q, h_kv, hd, B, shared, contig, q_scale, max_suffix):
    rng = np.random.default_rng(B * 31 + shared + hd + max_suffix)
    suffix = [int(x) for x in rng.integers(1, max_suffix, B)]   # >= 1: the new token is per-request
    lens = [shared + s for s in suffix]
    S = shared + sum(suffix) + 64
    free = np.arange(1, S) if contig else rng.permutation(np.arange(1, S))
    pre = free[:shared]
    stride = max(lens) + 4
    rtt = np.zeros((B, stride), dtype=np.int32)
    new = np.zeros(B, dtype=np.int32)
    off = shared
    for b, L in enumerate(lens):
        rtt[b, :shared] = pre
        n_own = L - shared
        rtt[b, shared:L - 1] = free[off:off + n_own - 1]
        new[b] = free[off + n_own - 1]
        off += n_own
    kpool = _vals(rng, S, h_kv, KIND_K, hd)
    vpool = _vals(rng, S, h_kv, KIND_V, hd)
    q = _vals(rng, B, h_q, KIND_Q, hd, scale=q_scale).cuda()
    kn = _vals(rng, B, h_kv, KIND_K, hd)
    vn = _vals(rng, B, h_kv, KIND_V, hd)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    new_d = torch.from_numpy(new).cuda()
    ws = torch.zeros(rx.rx_decode_cascade_workspace_bytes(cfg, B, max(lens), shared) + 1, dtype=torch.uint8,
                     device="cuda")
    kp, vp, rtt_d = kpool.cuda(), vpool.cuda(), torch.from_numpy(rtt).cuda()
    o = torch.full((B, h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    rx.rx_decode_cascade_append(cfg, rtt_d, None, seq, max(lens), shared, q, kn.cuda(), vn.cuda(), new_d, kp, vp, o, ws)
    # reference path for the append side effects
    kp2, vp2, rtt2 = kpool.cuda(), vpool.cuda(), torch.from_numpy(rtt).cuda()
    o2 = torch.empty_like(o)
    ws2 = torch.zeros(rx.rx_decode_workspace_bytes(cfg, B, max(lens)) + 1, dtype=torch.uint8, device="cuda")
    rx.rx_decode_append(cfg, rtt2, None, seq, max(lens), q, kn.cuda(), vn.cuda(), new_d, kp2, vp2, o2, ws2)
    torch.cuda.synchronize()
    assert torch.equal(kp, kp2) and torch.equal(vp, vp2) and torch.equal(rtt_d, rtt2)
    pool = A.OraclePool(S, h_kv, hd)
    pool.store(np.arange(S), kpool.float().numpy(), vpool.float().numpy())
    pool.store(new, kn.float().numpy(), vn.float().numpy())
    rows = [rtt[b].copy() for b in range(B)]
    for b, L in enumerate(lens):
        rows[b][L - 1] = new[b]
    ref = A.decode(pool, rows, lens, q.float().cpu().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
    _cmp(o, ref, f"cascade {h_q}/{h_kv}/{hd} B={B} shared={shared}")
    assert (o.float() - o2.float()).abs().max().item() <= 2e-2


def _decode_append_check(h_q, h_kv, hd, lens):
    """rx_decode_append == rx_store_kv + rtt append + rx_decode, bit for bit (pool, table, output)."""
    rng = np.random.default_rng(sum(lens))
    B = len(lens)
    S = sum(lens) + 64
    kp = _vals(rng, S, h_kv, KIND_K, hd).cuda()
    vp = _vals(rng, S, h_kv, KIND_V, hd).cuda()
    stride = max(lens) + 4
    perm = rng.permutation(np.arange(1, S))
    rtt = np.zeros((B, stride), dtype=np.int32)
    new = np.zeros(B, dtype=np.int32)
    off = 0
    for b, L in enumerate(lens):
        rtt[b, :L - 1] = perm[off:off + L - 1]
        new[b] = perm[off + L - 1]
        off += L
    q = _vals(rng, B, h_q, KIND_Q, hd).cuda()
    kn = _vals(rng, B, h_kv, KIND_K, hd).cuda()
    vn = _vals(rng, B, h_kv, KIND_V, hd).cuda()
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    seq = torch.tensor(lens, dtype=torch.int32, device="cuda")
    ws = torch.zeros(rx.rx_decode_workspace_bytes(cfg, B, max(lens)) + 1, dtype=torch.uint8, device="cuda")
    new_d = torch.from_numpy(new).cuda()
    # path 1: store + decode
    kp1, vp1, rtt1 = kp.clone(), vp.clone(), torch.from_numpy(rtt).cuda()
    idx = torch.tensor([b * stride + L - 1 for b, L in enumerate(lens)], dtype=torch.int64, device="cuda")
    rx.rx_store_kv(cfg, new_d, kn, vn, kp1, vp1, rtt1, idx)
    o1 = torch.empty((B, h_q, hd), dtype=torch.bfloat16, device="cuda")
    rx.rx_decode(cfg, rtt1, None, seq, max(lens), q, kp1, vp1, o1, ws)
    # path 2: fused
    kp2, vp2, rtt2 = kp.clone(), vp.clone(), torch.from_numpy(rtt).cuda()
    o2 = torch.empty_like(o1)
    rx.rx_decode_append(cfg, rtt2, None, seq, max(lens), q, kn, vn, new_d, kp2, vp2, o2, ws)
    torch.cuda.synchronize()
    assert torch.equal(kp1, kp2) and torch.equal(vp1, vp2) and torch.equal(rtt1, rtt2)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("h_q,h_kv,hd,B,shared,max_pre_own,max_ext", [
    (32, 32, 128, 12, 700, 200, 20),     # G=1, up to 3 column tiles, shared 700 (not a tile multiple)
    (32, 8, 128, 40, 1024, 90, 8),       # G=4
    (64, 8, 128, 24, 300, 50, 4),        # G=8
    (8, 2, 64, 80, 129, 40, 8),          # hd 64
])
@pytest.mark.parametrize("q_scale", [1.0, 4.0])
def test_extend_cascade_vs_oracle(h_q, h_kv, hd, B, shared, max_pre_own, max_ext, q_scale):
    """rx_extend_cascade: rows of B requests that share cached positions [0, shared) (same slots)
    plus their own cached tokens and a short new segment: shared part once on tcgen05, own part on
    the multi-query decode kernel, LSE merge — against the fp64 oracle, every row."""
    rng = np.random.default_rng(B + shared + hd)
    own = [int(x) for x in rng.integers(0, max_pre_own + 1, B)]
    ext = [int(x) for x in rng.integers(1, max_ext + 1, B)]
    ext[0] = max_ext
    pre = [shared + o_ for o_ in own]
    S = shared + sum(own) + sum(ext) + 64
    stride = max(p + e for p, e in zip(pre, ext)) + 5
    free = list(rng.permutation(np.arange(1, S)))
    rtt = np.zeros((B, stride), dtype=np.int32)
    sh_slots = free[:shared]
    off = shared
    for b in range(B):
        rtt[b, :shared] = sh_slots
        n = own[b] + ext[b]
        rtt[b, shared:shared + n] = free[off:off + n]
        off += n
    kpool = _vals(rng, S, h_kv, KIND_K, hd)
    vpool = _vals(rng, S, h_kv, KIND_V, hd)
    N = sum(ext)
    q = _vals(rng, N, h_q, KIND_Q, hd, scale=q_scale)
    kn = _vals(rng, N, h_kv, KIND_K, hd)
    vn = _vals(rng, N, h_kv, KIND_V, hd)
    indptr = np.concatenate([[0], np.cumsum(ext)]).astype(np.int32)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    kp, vp = kpool.cuda(), vpool.cuda()
    o = torch.full((N, h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda")
    ws = torch.zeros(rx.rx_extend_cascade_workspace_bytes(cfg, N, shared), dtype=torch.uint8, device="cuda")
    rows = torch.arange(B, dtype=torch.int32, device="cuda")
    rx.rx_extend_cascade(cfg, torch.from_numpy(rtt).cuda(), rows, torch.tensor(pre, dtype=torch.int32, device="cuda"),
                         torch.tensor(ext, dtype=torch.int32, device="cuda"), torch.from_numpy(indptr).cuda(), N,
                         max(ext), max(pre), shared, q.cuda(), kn.cuda(), vn.cuda(), kp, vp, o, ws)
    torch.cuda.synchronize()
    assert rx.rx_last_launch_count() == 4                      # the cascade path ran (store, suffix, shared, merge)
    pool = A.OraclePool(S, h_kv, hd)
    pool.store(np.arange(S), kpool.float().numpy(), vpool.float().numpy())
    ref = A.extend(pool, [rtt[b] for b in range(B)], pre, ext, q.float().numpy(), kn.float().numpy(),
                   vn.float().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
    _cmp(o, ref, f"extend_cascade {h_q}/{h_kv}/{hd} B={B} shared={shared}")
    for b in range(B):
        s_new = torch.from_numpy(rtt[b, pre[b]:pre[b] + ext[b]].astype(np.int64)).cuda()
        assert torch.equal(kp[s_new], kn[indptr[b]:indptr[b + 1]].cuda())


def test_concurrent_extends_on_two_streams():
    """Reentrancy (include/rx.h "Streams and concurrency"): two rx_extend calls with different
    workspaces run concurrently on two streams of one device — each persistent grid hands out its
    own work items from its own workspace header — and both match the oracle; their workspace
    headers are zero again afterwards.  Repeated so the grids overlap in time."""
    rng = np.random.default_rng(77)
    h_q, h_kv, hd = 32, 8, 128
    cases = []
    for c in range(2):
        B = 12
        pre = [int(x) for x in rng.integers(0, 900, B)]
        ext = [int(x) for x in rng.integers(100, 400, B)]
        S = sum(pre) + sum(ext) + 64
        rtt = np.zeros((B, max(p + e for p, e in zip(pre, ext))), dtype=np.int32)
        perm = rng.permutation(np.arange(1, S))
        off = 0
        for b in range(B):
            rtt[b, :pre[b] + ext[b]] = perm[off:off + pre[b] + ext[b]]
            off += pre[b] + ext[b]
        N = sum(ext)
        d = dict(pre=pre, ext=ext, rtt=rtt, N=N, S=S,
                 kpool=_vals(rng, S, h_kv, KIND_K, hd), vpool=_vals(rng, S, h_kv, KIND_V, hd),
                 q=_vals(rng, N, h_q, KIND_Q, hd), kn=_vals(rng, N, h_kv, KIND_K, hd),
                 vn=_vals(rng, N, h_kv, KIND_V, hd),
                 indptr=np.concatenate([[0], np.cumsum(ext)]).astype(np.int32))
        cases.append(d)
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    dev = []
    for d in cases:
        dev.append(dict(rtt=torch.from_numpy(d["rtt"]).cuda(), pre=torch.tensor(d["pre"], dtype=torch.int32).cuda(),
                        ext=torch.tensor(d["ext"], dtype=torch.int32).cuda(), ind=torch.from_numpy(d["indptr"]).cuda(),
                        q=d["q"].cuda(), kn=d["kn"].cuda(), vn=d["vn"].cuda(), kp=d["kpool"].cuda(),
                        vp=d["vpool"].cuda(),
                        o=torch.full((d["N"], h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda"),
                        ws=torch.zeros(rx.rx_extend_workspace_bytes(cfg, len(d["pre"]), max(d["ext"])),
                                       dtype=torch.uint8, device="cuda")))
    torch.cuda.synchronize()
    for _ in range(20):
        for d, x, st in zip(cases, dev, streams):
            rx.rx_extend(cfg, x["rtt"], None, x["pre"], x["ext"], x["ind"], d["N"], max(d["ext"]), max(d["pre"]),
                         x["q"], x["kn"], x["vn"], x["kp"], x["vp"], x["o"], x["ws"], stream=st)
    torch.cuda.synchronize()
    for d, x in zip(cases, dev):
        assert int(x["ws"].count_nonzero()) == 0
        pool = A.OraclePool(d["S"], h_kv, hd)
        pool.store(np.arange(d["S"]), d["kpool"].float().numpy(), d["vpool"].float().numpy())
        ref = A.extend(pool, [d["rtt"][b] for b in range(len(d["pre"]))], d["pre"], d["ext"], d["q"].float().numpy(),
                       d["kn"].float().numpy(), d["vn"].float().numpy(), h_q, h_kv, 1 / math.sqrt(hd))
        _cmp(x["o"], ref, "concurrent extend")


@pytest.mark.parametrize("h_q,h_kv,hd,shared", [(64, 8, 128, 2048), (32, 32, 128, 0), (8, 2, 64, 300)])
def test_decode_run_equals_per_step_calls(h_q, h_kv, hd, shared):
    """rx_decode_run (a run of decode steps in one library call, records read from one staged
    device array) is bit-identical to the same steps issued one rx_decode_cascade_append /
    rx_decode_append call at a time: outputs, pool rows and table entries."""
    rng = np.random.default_rng(h_q + shared)
    B, steps = 12, 5
    L0 = shared + 40
    stride = L0 + 20 + steps + 4
    S = shared + B * (stride - shared) + 64
    kp0 = _vals(rng, S, h_kv, KIND_K, hd).cuda()
    vp0 = _vals(rng, S, h_kv, KIND_V, hd).cuda()
    rtt0 = np.zeros((B, stride), dtype=np.int32)
    rtt0[:, :shared] = np.arange(1, shared + 1)
    own = (shared + 1 + np.arange(B * (stride - shared))).reshape(B, stride - shared).astype(np.int32)
    lens0 = L0 + rng.integers(0, 20, B)
    for b in range(B):
        rtt0[b, shared:lens0[b] - 1] = own[b, :lens0[b] - 1 - shared]
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    rows = np.arange(B, dtype=np.int32)[::-1].copy()            # batch entry b uses table row B-1-b
    recs, offs, maxs, qs, ks, vs = [], [], [], [], [], []
    off = 0
    for t in range(steps):
        seq = (lens0[rows] + t).astype(np.int32)
        new = own[rows, seq - 1 - shared].astype(np.int32)
        stable = np.full(B, L0 - 1, dtype=np.int32)
        recs.append(np.concatenate([new, seq, rows, stable]))
        offs.append(off)
        off += 4 * B
        maxs.append(int(seq.max()))
        qs.append(_vals(rng, B, h_q, KIND_Q, hd).cuda())
        ks.append(_vals(rng, B, h_kv, KIND_K, hd).cuda())
        vs.append(_vals(rng, B, h_kv, KIND_V, hd).cuda())
    rec = torch.from_numpy(np.concatenate(recs)).cuda()
    need = max(rx.rx_decode_cascade_workspace_bytes(cfg, B, stride, shared) if shared else 0,
               rx.rx_decode_workspace_bytes(cfg, B, stride))
    outs = []
    for mode in ("run", "steps"):
        kp, vp, rtt = kp0.clone(), vp0.clone(), torch.from_numpy(rtt0).cuda()
        ws = torch.zeros(need + 1, dtype=torch.uint8, device="cuda")
        o = [torch.full((B, h_q, hd), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(steps)]
        if mode == "run":
            rx.rx_decode_run(cfg, rtt, rec, offs, [B] * steps, maxs, shared, qs, ks, vs, kp, vp, o, ws)
            assert rx.rx_last_launch_count() >= steps
        else:
            for t in range(steps):
                d = rec[offs[t]:offs[t] + 4 * B]
                if shared:
                    rx.rx_decode_cascade_append(cfg, rtt, d[2 * B:3 * B], d[B:2 * B], maxs[t], shared, qs[t], ks[t],
                                                vs[t], d[:B], kp, vp, o[t], ws, stable_lens=d[3 * B:])
                else:
                    rx.rx_decode_append(cfg, rtt, d[2 * B:3 * B], d[B:2 * B], maxs[t], qs[t], ks[t], vs[t], d[:B],
                                        kp, vp, o[t], ws, stable_lens=d[3 * B:])
        torch.cuda.synchronize()
        outs.append((o, kp, vp, rtt))
    (o1, kp1, vp1, r1), (o2, kp2, vp2, r2) = outs
    assert torch.equal(kp1, kp2) and torch.equal(vp1, vp2) and torch.equal(r1, r2)
    for a, b in zip(o1, o2):
        assert torch.equal(a, b)
    assert all(torch.isfinite(a.float()).all() for a in o1)
