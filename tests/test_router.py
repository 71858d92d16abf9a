"""Data-parallel router (rx_router_*, App. A.4) —
C++ meta-tree against the oracle's per-token trie, the SPEC examples, and the
quiescent-convergence property with real worker trees (library rx_cache)
reporting evictions through rx_evict_paths."""
import random

import numpy as np
import pytest

from oracle.router import OracleRouter
from paper_2312_07104_b200.api import Router, RadixCache


def test_spec_cold_start_round_robin():          # S:442 [DERIVED]
    r = Router(4)
    loads = np.zeros(4, dtype=np.int64)
    reqs = [np.arange(1, 9) + 100 * i for i in range(8)]
    w, a = r.rx_router_dispatch(reqs, loads, 0.0)
    assert list(w) == [0, 1, 2, 3, 0, 1, 2, 3] and list(a) == [0] * 8


def test_spec_unique_affinity():                  # S:443 [TRIVIAL]
    r = Router(4)
    r.rx_router_insert(2, [5, 6, 7, 8])
    loads = np.zeros(4, dtype=np.int64)
    w, a = r.rx_router_dispatch([[5, 6, 7, 8, 9]], loads, 0.0)
    assert list(w) == [2] and list(a) == [4]


def test_spec_eviction_sync():
    r = Router(2)
    r.rx_router_insert(1, [1, 2, 3, 4])
    assert r.rx_router_sync() == 0                   # empty queue
    r.rx_router_queue_evict(1, [1, 2, 3, 4], 0)      # worker 1 evicts its only cached path
    assert list(r.rx_router_affinity([1, 2, 3])) == [0, 3]   # stale until synced
    assert r.rx_router_sync() == 1
    assert list(r.rx_router_affinity([1, 2, 3])) == [0, 0]
    assert r.rx_router_dump_json()["children"] == []


def test_few_shot_balanced_with_load_weight():
    """MMLU-like batch (shared few-shot prefix): with load_weight 1 every worker
    gets the prefix once and the batch spreads evenly (P:638 'linear scaling and
    an optimal cache hit rate')."""
    rng = np.random.default_rng(0)
    pre = rng.integers(1, 30000, 1500)
    reqs = [np.concatenate([pre, rng.integers(1, 30000, 60)]) for _ in range(64)]
    r = Router(4)
    loads = np.zeros(4, dtype=np.int64)
    w, a = r.rx_router_dispatch(reqs, loads, 1.0)
    counts = np.bincount(w, minlength=4)
    assert counts.min() >= 14 and counts.max() <= 18
    assert (a == 0).sum() == 4                        # exactly one cold prefix per worker
    # pure affinity keeps the whole group on one worker
    r2 = Router(4)
    l2 = np.zeros(4, dtype=np.int64)
    w2, _ = r2.rx_router_dispatch(reqs, l2, 0.0)
    assert len(set(w2.tolist())) == 1


@pytest.mark.parametrize("seed", range(6))
def test_router_vs_oracle(seed):
    rng = random.Random(seed)
    W = rng.choice([2, 3, 4, 8])
    c, o = Router(W), OracleRouter(W)
    lc = np.zeros(W, dtype=np.int64)
    lo = [0] * W
    known = []
    for step in range(120):
        op = rng.random()
        if op < 0.4:
            batch = []
            for _ in range(rng.randrange(1, 6)):
                if known and rng.random() < 0.6:
                    base = rng.choice(known)
                    batch.append(base[:rng.randrange(1, len(base) + 1)] + [rng.randrange(1, 5) for _ in range(rng.randrange(0, 4))])
                else:
                    batch.append([rng.randrange(1, 5) for _ in range(rng.randrange(1, 8))])
            lw = rng.choice([0.0, 0.5, 1.0, 3.0])
            wc, ac = c.rx_router_dispatch([np.array(b) for b in batch], lc, lw)
            wo, ao = o.dispatch(batch, lo, lw)
            assert list(wc) == wo and list(ac) == ao and list(lc) == lo, step
            known.extend(batch)
        elif op < 0.6 and known:
            w = rng.randrange(W)
            t = rng.choice(known)
            c.rx_router_insert(w, t)
            o.insert(w, t)
        elif op < 0.85 and known:
            w = rng.randrange(W)
            t = rng.choice(known)
            ls = rng.randrange(0, len(t))
            c.rx_router_queue_evict(w, t, ls)
            o.queue_evict(w, t, ls)
        else:
            assert c.rx_router_sync() == o.sync()
        for _ in range(3):
            q = rng.choice(known) if known else [1]
            assert list(c.rx_router_affinity(q)) == o.affinity(q)


def test_quiescent_convergence_with_worker_trees():
    """Workers = library rx_cache trees; every insert and every eviction (rx_evict_paths)
    is reported.  After the queue drains, affinity[w] == worker w's match_prefix length."""
    rng = random.Random(7)
    W = 3
    router = Router(W)
    workers = [RadixCache(60) for _ in range(W)]
    seqs = []
    for it in range(300):
        w = rng.randrange(W)
        t = ([rng.randrange(1, 4) for _ in range(rng.randrange(1, 9))] if not seqs or rng.random() < 0.5
             else rng.choice(seqs)[:rng.randrange(1, 8)] + [rng.randrange(1, 4) for _ in range(rng.randrange(1, 4))])
        seqs.append(t)
        tree = workers[w]
        node, m, pre = tree.rx_match_prefix(t)
        need = len(t) - m
        s = tree.rx_alloc(need)
        if s is None:
            ev, paths = tree.rx_evict_paths(need - tree.rx_available())
            for path, leaf_start, _ in paths:
                router.rx_router_queue_evict(w, path, leaf_start)
            s = tree.rx_alloc(need)
            if s is None:
                continue
        tree.rx_insert(t, list(pre) + list(s))
        router.rx_router_insert(w, t)
        if rng.random() < 0.2:
            router.rx_router_sync()
    router.rx_router_sync()
    for q in seqs[-80:]:
        aff = router.rx_router_affinity(q)
        for w in range(W):
            _, m, _ = workers[w].rx_match_prefix(q)
            assert aff[w] == m, (q, w, aff, m)
