"""Theorem 1 (§3, proof P:578-618) as a pin for both trees.

For a batch of requests whose radix tree T has edges e, any order computes at
least C = sum_e |e| prefill tokens; with a cache of capacity >= the longest
request, the longest-shared-prefix-first (LSPF) order — re-match every
waiting request, run the one with the longest match — reaches exactly C, so
its hit rate is 1 - C / sum(prompt tokens), and no permutation
(brute force, <= 6 requests) does better.  Outputs are empty.
"""
import itertools
import random

import pytest

from oracle.radix import RadixCache as OracleCache
from paper_2312_07104_b200 import RadixCache as LibCache


class _O:
    def __init__(self, n):
        self.t = OracleCache(n)

    def match(self, x):
        node, m, _ = self.t.match_prefix(x)
        return node, m

    def run(self, x, node, m):
        self.t.inc_ref(node)
        s = self.t.alloc(len(x) - m)
        if s is None:
            self.t.evict(len(x) - m - self.t.available())
            s = self.t.alloc(len(x) - m)
        assert s is not None
        _, _, pre = self.t.match_prefix(x[:m]) if m else (None, 0, [])
        self.t.dec_ref(node)
        self.t.insert(x, list(pre) + list(s))


class _L:
    def __init__(self, n):
        self.t = LibCache(n)

    def match(self, x):
        node, m, _ = self.t.rx_match_prefix(x)
        return node, m

    def run(self, x, node, m):
        self.t.rx_inc_ref(node)
        s = self.t.rx_alloc(len(x) - m)
        if s is None:
            self.t.rx_evict(len(x) - m - self.t.rx_available())
            s = self.t.rx_alloc(len(x) - m)
        assert s is not None
        _, _, pre = self.t.rx_match_prefix(x[:m]) if m else (None, 0, [])
        self.t.rx_dec_ref(node)
        self.t.rx_insert(x, list(pre) + list(s))


def _random_batch(rng, n_req):
    """Requests from a random token tree; no request is a prefix of another."""
    reqs = []
    while len(reqs) < n_req:
        base = reqs[rng.randrange(len(reqs))] if reqs and rng.random() < 0.7 else []
        cut = rng.randrange(0, len(base) + 1) if base else 0
        tail = [rng.randrange(1, 6) for _ in range(rng.randrange(1, 5))]
        r = base[:cut] + tail
        if any(r == q[:len(r)] or q == r[:len(q)] for q in reqs):
            continue
        reqs.append(r)
    return reqs


def _edge_sum(reqs):
    """sum of edge lengths of the radix tree of reqs = number of distinct non-empty prefixes."""
    return len({tuple(r[:i]) for r in reqs for i in range(1, len(r) + 1)})


def _computed_in_order(make, reqs, order, cap):
    t = make(cap)
    total = 0
    for i in order:
        node, m = t.match(reqs[i])
        total += len(reqs[i]) - m
        t.run(reqs[i], node, m)
    return total


def _computed_lspf(make, reqs, cap):
    t = make(cap)
    waiting = list(range(len(reqs)))
    total = 0
    while waiting:
        best = None
        for i in waiting:
            node, m = t.match(reqs[i])
            if best is None or m > best[1]:
                best = (i, m, node)
        i, m, node = best
        total += len(reqs[i]) - m
        t.run(reqs[i], node, m)
        waiting.remove(i)
    return total


@pytest.mark.parametrize("make", [_O, _L])
@pytest.mark.parametrize("seed", range(12))
def test_theorem1_lspf_optimal(make, seed):
    rng = random.Random(seed)
    reqs = _random_batch(rng, rng.randrange(3, 7))
    cap = max(len(r) for r in reqs) + 1               # + the reserved padding slot
    C = _edge_sum(reqs)
    lspf = _computed_lspf(make, reqs, cap)
    assert lspf == C
    brute = min(_computed_in_order(make, reqs, p, cap) for p in itertools.permutations(range(len(reqs))))
    assert brute == C
    total = sum(len(r) for r in reqs)
    hit = 1 - lspf / total
    assert hit == pytest.approx(1 - C / total)


def test_theorem1_bound_is_tight_only_with_enough_capacity():
    """The lower bound holds for every order and capacity; a bad order can exceed it."""
    rng = random.Random(99)
    worse = 0
    for _ in range(20):
        reqs = _random_batch(rng, 5)
        cap = max(len(r) for r in reqs) + 1
        C = _edge_sum(reqs)
        for p in itertools.permutations(range(len(reqs))):
            c = _computed_in_order(_O, reqs, p, cap)
            assert c >= C
            worse += c > C
    assert worse > 0
