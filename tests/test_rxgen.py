"""Pins for the seeded input generator (rxgen): published splitmix64 values and
agreement of its three independent forms."""
import numpy as np
import torch

from rxgen.hashing import splitmix64_int, splitmix64_np, splitmix64_t, prefix_hashes, next_token
from rxgen.values import gen_values, gen_values_np, KIND_K, KIND_V, KIND_Q
from rxgen import workloads


def test_splitmix64_published_values():
    # splitmix64 stream seeded with 0: first outputs are the published test vector
    # (Vigna's reference splitmix64.c; e.g. used to seed xoshiro).
    assert splitmix64_int(0) == 0xE220A8397B1DCDAF
    # second output of that stream = mix(2*GOLDEN)
    assert splitmix64_int(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_splitmix64_forms_agree():
    rng = np.random.default_rng(1)
    x = rng.integers(0, 2**63, 20000, dtype=np.uint64) * np.uint64(3)
    a = splitmix64_np(x)
    b = splitmix64_t(torch.from_numpy(x.view(np.int64))).numpy().view(np.uint64)
    assert np.array_equal(a, b)
    for v, w in zip(x[:200].tolist(), a[:200].tolist()):
        assert splitmix64_int(v) == w


def test_gen_values_torch_equals_numpy():
    h = prefix_hashes(list(range(1, 300)), 7)
    for kind, scale in ((KIND_K, 1.0), (KIND_V, 1.0), (KIND_Q, 4.0)):
        t = gen_values(h, [0, 5, 31], kind, 128, scale=scale).float().numpy()
        n = gen_values_np(h, [0, 5, 31], kind, 128, scale=scale)
        assert np.array_equal(t, n)


def test_gen_values_distribution():
    h = np.arange(4096, dtype=np.uint64)
    v = gen_values(h, range(4), KIND_K, 64).float()
    assert abs(v.mean().item()) < 0.01
    assert abs(v.std().item() - 1.0) < 0.01
    assert v.abs().max().item() <= 3.47
    # values are bf16: round-trip exact
    assert torch.equal(v.to(torch.bfloat16).float(), v)


def test_prefix_hash_depends_only_on_prefix():
    a = prefix_hashes([5, 6, 7, 8], 3)
    b = prefix_hashes([5, 6, 9, 8], 3)
    assert np.array_equal(a[:2], b[:2]) and not np.array_equal(a[2:], b[2:])
    assert 1 <= next_token(int(a[-1]), 32000) < 32000


def test_workload_shapes():
    w = workloads.c1()
    assert w.shape.h_q == 8 and w.shape.h_kv == 2 and w.shape.head_dim == 64
    assert len(w.phases[1][1]) == 16 and len(w.phases[1][1][0].prompt) == 96
    w5 = workloads.c5(n_req=4, prefix=64)
    assert w5.shape.group == 8
    w4 = workloads.c4()
    assert sum(len(l) for l in w4.meta["levels"]) == 4 + 16 + 64
