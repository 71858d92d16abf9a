"""librx host half (C++ radix tree + slot pool) against the oracle — CPU only.

* the library loads and exports every function include/rx.h declares;
* the Fig. 3 golden trace and the SPEC examples hold on the C++ tree;
* random op sequences replayed on both trees give bit-identical results
  (matched lengths, slot vectors, ref deltas, eviction runs in order, insert
  results, full pre-order dumps with ids and LRU stamps).
"""
import random
import re
import os

import numpy as np
import pytest

from oracle.radix import RadixCache as OracleCache, Underflow
from paper_2312_07104_b200 import RadixCache, RxError
from paper_2312_07104_b200._lib import lib, SIGNATURES
from tree_common import run_fig3

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "rx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(rx_[a-z0-9_]+)\s*\(", src))
    return names


def test_exports_every_declared_symbol():
    names = _header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert names == set(SIGNATURES), names ^ set(SIGNATURES)
    assert b"sm_100a" in lib.rx_version()


class LibAdapter:
    def __init__(self, n):
        self.t = RadixCache(n)

    def match(self, toks):
        return self.t.rx_match_prefix(toks)

    def inc(self, h):
        return self.t.rx_inc_ref(h)

    def dec(self, h):
        return self.t.rx_dec_ref(h)

    def evict(self, k):
        n, runs = self.t.rx_evict(k)
        return n, [list(r) for r in runs]

    def alloc(self, n):
        s = self.t.rx_alloc(n)
        assert s is not None
        return list(s)

    def insert(self, toks, slots):
        return self.t.rx_insert(toks, slots)

    def dump(self):
        return self.t.rx_dump_json()


def _check(ok, msg):
    assert ok, msg


def test_fig3_golden_trace_lib():
    run_fig3(LibAdapter(1000), _check)


def test_spec_examples_lib():
    t = RadixCache(100)
    node, m, s = t.rx_match_prefix([5, 6, 7])
    assert (node, m, len(s)) == (0, 0, 0)
    assert t.rx_insert([1, 2, 3], t.rx_alloc(3)) == (3, 0)
    assert t.rx_insert([1, 2, 3], t.rx_alloc(3)) == (0, 3)
    assert t.rx_insert([1, 2, 4, 5], t.rx_alloc(4)) == (2, 2)
    node, m, s = t.rx_match_prefix([1, 2, 3])
    assert m == 3 and list(s) == [1, 2, 3]
    assert t.rx_inc_ref(node) == -3           # [1,2] and [3] newly pinned
    assert t.rx_inc_ref(node) == 0
    assert t.rx_dec_ref(node) == 0
    assert t.rx_dec_ref(node) == 3
    with pytest.raises(RxError) as e:
        t.rx_dec_ref(node)
    assert e.value.status == -3                # RX_E_UNDERFLOW
    ev, runs = t.rx_evict(100)
    assert ev == 5 and t.rx_total_cached() == 0
    with pytest.raises(RxError) as e:
        t.rx_inc_ref(node)
    assert e.value.status == -4                # RX_E_STALE


def test_alloc_free_errors():
    t = RadixCache(8)
    assert list(t.rx_alloc(3)) == [1, 2, 3]
    t.rx_free([2])
    assert list(t.rx_alloc(2)) == [2, 4]
    assert t.rx_alloc(10) is None and t.rx_available() == 3
    with pytest.raises(RxError):
        t.rx_free([5])          # already free
    with pytest.raises(RxError):
        t.rx_free([0])          # reserved
    with pytest.raises(RxError):
        t.rx_free([1, 1])       # duplicate
    assert t.rx_available() == 3


def test_alloc_bitmap_large_pool():
    n = 1 << 20
    t = RadixCache(n)
    a = t.rx_alloc(300000)
    assert a[0] == 1 and a[-1] == 300000 and np.all(np.diff(a) == 1)
    t.rx_free(a[1000:2000:3])
    freed = a[1000:2000:3]                      # 334 slots
    b = t.rx_alloc(400)
    expect = np.concatenate([freed, np.arange(300001, 300001 + 400 - len(freed))])
    assert np.array_equal(b, expect)
    assert t.rx_available() == n - 1 - 300000 - (400 - len(freed))


def _replay(seed, n_ops, alphabet, maxlen, slots):
    rng = random.Random(seed)
    o = OracleCache(slots)
    c = RadixCache(slots)
    pinned = []
    for step in range(n_ops):
        op = rng.random()
        toks = [rng.randrange(1, alphabet + 1) for _ in range(rng.randrange(1, maxlen + 1))]
        if op < 0.35:
            on, om, os_ = o.match_prefix(toks)
            cn, cm, cs = c.rx_match_prefix(toks)
            assert (om, list(os_)) == (cm, list(cs)) and on.id == cn, step
            if rng.random() < 0.35:
                assert o.inc_ref(on) == c.rx_inc_ref(cn)
                pinned.append((on, cn))
        elif op < 0.7:
            on, om, os_ = o.match_prefix(toks)
            cn, cm, cs = c.rx_match_prefix(toks)
            assert om == cm and list(os_) == list(cs)
            need = len(toks) - om
            if rng.random() < 0.3 and om:
                need = len(toks)          # recompute the prefix: duplicate slots
            sa = o.alloc(need)
            sb = c.rx_alloc(need)
            assert (sa is None) == (sb is None)
            if sa is None:
                ev_o = o.evict(need - o.available())
                ev_c = c.rx_evict(need - c.rx_available())
                assert ev_o[0] == ev_c[0] and ev_o[1] == [list(r) for r in ev_c[1]]
                sa = o.alloc(need)
                sb = c.rx_alloc(need)
                assert (sa is None) == (sb is None)
                if sa is None:
                    continue
            assert list(sa) == list(sb)
            full = (list(os_) + list(sa)) if need == len(toks) - om else list(sa)
            assert o.insert(toks, full) == c.rx_insert(toks, full)
        elif op < 0.85 and pinned:
            on, cn = pinned.pop(rng.randrange(len(pinned)))
            assert o.dec_ref(on) == c.rx_dec_ref(cn)
        else:
            k = rng.randrange(0, 12)
            ev_o = o.evict(k)
            ev_c = c.rx_evict(k)
            assert ev_o[0] == ev_c[0] and ev_o[1] == [list(r) for r in ev_c[1]], step
        assert o.evictable_size() == c.rx_evictable_size()
        assert o.total_cached() == c.rx_total_cached()
        assert o.available() == c.rx_available()
        if step % 50 == 0:
            assert o.dump() == c.rx_dump_json()
    assert o.dump() == c.rx_dump_json()


@pytest.mark.parametrize("seed", range(10))
def test_replay_vs_oracle(seed):
    _replay(seed, 1500, alphabet=4, maxlen=8, slots=80)


def test_replay_vs_oracle_wide():
    _replay(123, 3000, alphabet=30, maxlen=40, slots=600)
