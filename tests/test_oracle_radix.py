"""Pins for the oracle radix tree (oracle/radix.py):

* SPEC.md worked examples, hand-simulated;
* the Fig. 3 caption: structure after every step and the
  eviction order of every step (tests/golden/fig3_radix_trace.json);
* brute force: a flat map {token prefix -> slot} maintained beside the tree
  must agree with match_prefix on random op sequences, plus the
  invariants of SPEC.md:158-164 (radix property, accounting, eviction safety,
  LRU-monotone eviction).
"""
import random

import pytest
from hypothesis import given, settings, strategies as st

from oracle.radix import RadixCache, Underflow
from tree_common import run_fig3


class OracleAdapter:
    def __init__(self, n):
        self.t = RadixCache(n)

    def match(self, toks):
        return self.t.match_prefix(toks)

    def inc(self, h):
        return self.t.inc_ref(h)

    def dec(self, h):
        return self.t.dec_ref(h)

    def evict(self, k):
        return self.t.evict(k)

    def alloc(self, n):
        s = self.t.alloc(n)
        assert s is not None
        return s

    def insert(self, toks, slots):
        return self.t.insert(toks, slots)

    def dump(self):
        return self.t.dump()


def _check(ok, msg):
    assert ok, msg


def test_fig3_golden_trace():
    run_fig3(OracleAdapter(1000), _check)


# ---------------------------------------------------------------- SPEC examples
def test_spec_match_empty():            # S:119 [TRIVIAL]
    t = RadixCache(100)
    node, m, slots = t.match_prefix([5, 6, 7])
    assert node is t.root and m == 0 and slots == []


def test_spec_match_split():            # S:120 [DERIVED]
    t = RadixCache(100)
    t.insert([1, 2, 3, 4], t.alloc(4))
    node, m, slots = t.match_prefix([1, 2, 9])
    assert m == 2 and node.tokens == [1, 2] and slots == [1, 2]
    assert [c.tokens for c in node.children.values()] == [[3, 4]]


def test_spec_insert_examples():
    t = RadixCache(100)
    assert t.insert([1, 2, 3], t.alloc(3)) == (3, 0)
    s = t.alloc(3)
    assert t.insert([1, 2, 3], s) == (0, 3)          # idempotent; passed slots freed (R10)
    assert t.insert([1, 2, 4, 5], t.alloc(4)) == (2, 2)
    top = t.root.children[1]
    assert top.tokens == [1, 2] and sorted(c.tokens[0] for c in top.children.values()) == [3, 4]


def test_spec_ref_examples():
    t = RadixCache(100)
    t.insert([1, 2, 3, 4], t.alloc(4))
    node, m, _ = t.match_prefix([1, 2, 3, 4])
    assert t.inc_ref(node) == -4
    assert t.inc_ref(node) == 0
    assert t.dec_ref(node) == 0
    assert t.dec_ref(node) == 4
    with pytest.raises(Underflow):
        t.dec_ref(node)


def test_spec_evict_lru():
    t = RadixCache(100)
    assert t.evict(0) == (0, [])
    t.insert([1, 2, 3, 4, 5], t.alloc(5))       # clock 1
    t.match_prefix([9])                          # clock 2 (no match)
    t.insert([7, 8, 9, 10, 11], t.alloc(5))      # clock 3
    t.match_prefix([7])                          # clock 4: refreshes [7..11]
    n, runs = t.evict(4)
    assert n == 5 and runs == [[1, 2, 3, 4, 5]]


def test_spec_evictable_size():
    t = RadixCache(100)
    assert t.evictable_size() == 0
    t.insert(list(range(1, 11)), t.alloc(10))
    assert t.evictable_size() == 10
    node, m, _ = t.match_prefix(list(range(1, 7)))
    t.inc_ref(node)
    assert m == 6 and t.evictable_size() == 4


def test_alloc_smallest_first_and_nomem():
    t = RadixCache(8)
    assert t.alloc(3) == [1, 2, 3]
    t.free_slots([2])
    assert t.alloc(2) == [2, 4]
    assert t.alloc(10) is None and t.available() == 3


def test_evict_exposes_parent_and_respects_pins():
    t = RadixCache(100)
    t.insert([1, 2, 3], t.alloc(3))
    t.insert([1, 2, 4], t.alloc(3))        # split: [1,2] -> {[3], [4]}
    node, _, _ = t.match_prefix([1, 2, 4])
    t.inc_ref(node)
    n, runs = t.evict(100)
    assert runs == [[3]] and n == 1        # [1,2] and [4] pinned
    t.dec_ref(node)
    n, runs = t.evict(100)
    assert runs == [[6], [1, 2]] and n == 3


# ---------------------------------------------------------------- brute force
def _brute_match(flat, toks):
    m = 0
    slots = []
    while m < len(toks) and tuple(toks[:m + 1]) in flat:
        slots.append(flat[tuple(toks[:m + 1])])
        m += 1
    return m, slots


def _check_invariants(t: RadixCache, flat):
    nodes = t._nodes()
    for n in nodes:
        firsts = [c.tokens[0] for c in n.children.values()]
        assert len(firsts) == len(set(firsts))                  # radix property
        for k, c in n.children.items():
            assert c.tokens[0] == k and c.parent is n and len(c.tokens) == len(c.slots) > 0
            assert n is t.root or n.ref >= c.ref                # pins propagate up
            assert n is t.root or n.last_access >= c.last_access  # stamps propagate up
    assert t.total_cached() == len(flat)                        # accounting
    assert 0 <= t.evictable_size() <= t.total_cached()
    cached = [s for n in nodes for s in n.slots]
    assert len(set(cached)) == len(cached)
    assert not (set(cached) & set(t.free))


def _random_ops(seed, n_ops, alphabet=4, maxlen=7, slots=60):
    rng = random.Random(seed)
    t = RadixCache(slots)
    flat = {}                 # token prefix -> slot
    slot_prefix = {}
    pinned = []               # (node, prefix tuple)
    for _ in range(n_ops):
        op = rng.random()
        toks = [rng.randrange(1, alphabet + 1) for _ in range(rng.randrange(1, maxlen + 1))]
        if op < 0.35:
            m, slots_b = _brute_match(flat, toks)
            node, m2, s2 = t.match_prefix(toks)
            assert (m2, s2) == (m, slots_b)
            if rng.random() < 0.3:
                t.inc_ref(node)
                pinned.append((node, tuple(toks[:m2])))
        elif op < 0.7:
            m, _ = _brute_match(flat, toks)
            new = t.alloc(len(toks) - m)
            if new is None:
                continue
            passed = [flat[tuple(toks[:i + 1])] for i in range(m)]
            # sometimes pass fresh (duplicate) slots for the cached part too
            if m and rng.random() < 0.3:
                dup = t.alloc(m)
                if dup is not None:
                    passed = dup
            slots = passed + new
            before_free = len(t.free)
            nc, nd = t.insert(toks, slots)
            assert nc == len(toks) - m
            for i in range(m, len(toks)):
                flat[tuple(toks[:i + 1])] = slots[i]
                slot_prefix[slots[i]] = tuple(toks[:i + 1])
            assert len(t.free) == before_free + nd
        elif op < 0.85 and pinned:
            node, pre = pinned.pop(rng.randrange(len(pinned)))
            t.dec_ref(node)
        else:
            k = rng.randrange(0, 10)
            pinned_prefixes = set()
            for _, pre in pinned:
                for i in range(1, len(pre) + 1):
                    pinned_prefixes.add(pre[:i])
            ev_before = t.evictable_size()
            n, runs = t.evict(k)
            assert n >= min(k, ev_before) and (n == 0 or n - max(len(r) for r in runs) < k)
            for run in runs:
                for s in run:
                    pre = slot_prefix.pop(s)
                    assert pre not in pinned_prefixes                   # eviction safety
                    del flat[pre]
        _check_invariants(t, flat)


@pytest.mark.parametrize("seed", range(8))
def test_random_ops_vs_flat_map(seed):
    _random_ops(seed, 1500)


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 10**9))
def test_random_ops_hypothesis(seed):
    _random_ops(seed, 200, alphabet=3, maxlen=6, slots=40)


def test_lru_monotone_eviction_order():
    """Within one evict call the stamps of removed nodes never decrease."""
    rng = random.Random(5)
    t = RadixCache(400)
    for i in range(60):
        toks = [rng.randrange(1, 4) for _ in range(rng.randrange(1, 8))]
        s = t.alloc(len(toks))
        if s is None:
            break
        t.insert(toks, s)
        if rng.random() < 0.5:
            t.match_prefix([rng.randrange(1, 4) for _ in range(3)])
    stamps = {tuple(n.slots): n.last_access for n in t._nodes() if n is not t.root}
    n, runs = t.evict(10**9)
    seq = [stamps[tuple(r)] for r in runs]
    assert t.total_cached() == 0 and len(runs) > 5
    assert seq == sorted(seq)
