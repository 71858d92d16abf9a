"""Cache-aware scheduling (Alg. 1 admission; §3; ablation P:432) in the
library (rx_schedule, C++) against the oracle driver's plain-Python admission, plus pins from the
paper that do not depend on either implementation:

* Theorem 1 (proof P:578-618): driving the order with rx_schedule's LSPF choice computes
  exactly sum_e |e| prefill tokens (the lower bound of any order) on random request trees;
* the ablation claim ("cache thrashing"): on an interleaved multi-prefix queue that
  does not fit the pool, LSPF's hit rate beats FCFS and random; FCFS thrashes to 0;
* the fit-check invariant (reading R25): after every admission sum(size) < evictable + free, so the
  batch's allocation never fails.
CPU only (plan pass: tree ops, no kernels)."""
import json
import random

import numpy as np
import pytest

from oracle.driver import OracleEngine
from oracle.radix import RadixCache as OracleCache
from paper_2312_07104_b200 import RadixCache as LibCache
from paper_2312_07104_b200._lib import RxError
from paper_2312_07104_b200.engine import Engine
from rxgen import sched_keys, workloads

from test_theorem1 import _edge_sum, _random_batch


def _hit(stats):
    return stats["cached_prompt_tokens"] / stats["prompt_tokens"]


def _both(wl, policy):
    o = OracleEngine(wl, policy=policy)
    o.run_workload()
    e = Engine(wl, plan_only=True, record=True, policy=policy)
    e.run_workload()
    return o, e


@pytest.mark.parametrize("policy", ["lspf", "fcfs", "random"])
@pytest.mark.parametrize("cfg", [
    lambda: workloads.mix(),
    lambda: workloads.mix(seed=3, groups=3, per_group=9, prefix=300, num_slots=900),
    lambda: workloads.c4(),
    lambda: workloads.c4(seed=1, root=300, p_lo=8, p_hi=40, t_lo=4, t_hi=20, capacity_frac=0.5),
])
def test_schedule_trace_equal(cfg, policy):
    o, e = _both(cfg(), policy)
    assert len(o.trace) == len(e.trace)
    for i, (x, y) in enumerate(zip(o.trace, e.trace)):
        assert x == y, f"trace entry {i}: oracle {str(x)[:200]} != lib {str(y)[:200]}"
    assert o.stats["cached_prompt_tokens"] == e.stats["cached_prompt_tokens"]


def test_ablation_lspf_beats_fcfs_and_random():
    """switching between unrelated requests thrashes the cache; LSPF keeps a group
    together.  The MIX queue interleaves 4 prefixes of 1024 tokens; the pool holds ~2."""
    wl = workloads.mix()
    hits = {p: _hit(_both(wl, p)[1].stats) for p in ("lspf", "fcfs", "random")}
    assert hits["lspf"] > hits["random"] > hits["fcfs"]
    assert hits["fcfs"] == 0.0
    # each prefix is computed at most a few times under LSPF: hit rate close to the
    # one-pass bound 1 - (groups * prefix + questions) / prompt tokens
    o = _both(wl, "lspf")[0]
    assert hits["lspf"] > 0.85


def _lib_lspf_computed(reqs, cap):
    """Theorem-1 harness with the order chosen by rx_schedule: each step, the first request it
    admits (its LSPF choice) runs; the other admitted requests are unpinned again."""
    t = LibCache(cap)
    waiting = list(range(len(reqs)))
    total = 0
    while waiting:
        toks = np.concatenate([np.asarray(reqs[i], np.int32) for i in waiting])
        off = np.zeros(len(waiting) + 1, np.int64)
        off[1:] = np.cumsum([len(reqs[i]) for i in waiting])
        nodes, matched, sl, adm, _ = t.rx_schedule(toks, off, [0] * len(waiting), "lspf")
        assert len(adm) >= 1
        b = int(adm[0])
        assert matched[b] == matched.max()                  # LSPF: the longest match goes first
        for k in adm[1:]:
            t.rx_dec_ref(int(nodes[k]))
        i = waiting[b]
        x, m = reqs[i], int(matched[b])
        total += len(x) - m
        s = t.rx_alloc(len(x) - m)
        if s is None:
            t.rx_evict(len(x) - m - t.rx_available())
            s = t.rx_alloc(len(x) - m)
        assert s is not None
        pre = sl[off[b]:off[b] + m]
        t.rx_dec_ref(int(nodes[b]))
        t.rx_insert(x, list(pre) + list(s))
        waiting.remove(i)
    return total


@pytest.mark.parametrize("seed", range(16))
def test_theorem1_via_rx_schedule(seed):
    rng = random.Random(1000 + seed)
    reqs = _random_batch(rng, rng.randrange(3, 9))
    # cache >= the longest request (Theorem 1) + the padding slot + 1 for Alg. 1's strict `<`
    cap = max(len(r) for r in reqs) + 2
    assert _lib_lspf_computed(reqs, cap) == _edge_sum(reqs)


def _oracle_admit(tree, prompts, max_new, policy, keys):
    """Alg. 1 P:526-547 with R7/R11/R25 written out on the oracle tree."""
    m = [tree.match_prefix(p) for p in prompts]
    idx = list(range(len(prompts)))
    if policy == "lspf":
        order = sorted(idx, key=lambda i: (-m[i][1], i))
    elif policy == "fcfs":
        order = idx
    else:
        order = sorted(idx, key=lambda i: (int(keys[i]), i))
    avail = tree.evictable_size() + tree.available()
    cur = 0
    adm = []
    for i in order:
        size = len(prompts[i]) - min(m[i][1], len(prompts[i]) - 1) + max_new[i]
        d = tree.inc_ref(m[i][0])
        if size + cur < avail + d:
            avail += d
            cur += size
            adm.append((i, d))
        else:
            tree.dec_ref(m[i][0])
    return [x[1] for x in m], adm, [x[0] for x in m]


@pytest.mark.parametrize("policy", ["lspf", "fcfs", "random"])
@pytest.mark.parametrize("seed", range(6))
def test_rx_schedule_random_steps(policy, seed):
    """Random op sequences: admission steps interleaved with inserts, finishes and evictions; every
    step's matched lengths, admitted order and deltas equal the oracle's, and the R25 invariant
    holds (the admitted sizes fit evictable + free after all pins)."""
    rng = np.random.default_rng(seed)
    cap = 400
    ot, lt = OracleCache(cap), LibCache(cap)
    pinned = []
    for step in range(30):
        B = int(rng.integers(1, 7))
        base = [rng.integers(1, 6, int(rng.integers(1, 40))).astype(np.int32) for _ in range(3)]
        prompts = [np.concatenate([base[int(rng.integers(0, 3))][:int(rng.integers(0, 40))],
                                   rng.integers(1, 6, int(rng.integers(1, 30))).astype(np.int32)]) for _ in range(B)]
        max_new = [int(rng.integers(0, 60)) for _ in range(B)]
        keys = sched_keys(seed, step, B)
        om, oadm, onodes = _oracle_admit(ot, [list(p) for p in prompts], max_new, policy, keys)
        off = np.zeros(B + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in prompts])
        nodes, matched, sl, adm, deltas = lt.rx_schedule(np.concatenate(prompts), off, max_new, policy,
                                                         keys if policy == "random" else None)
        assert list(matched) == om
        assert [int(a) for a in adm] == [a for a, _ in oadm]
        assert [int(d) for d in deltas] == [d for _, d in oadm]
        need = sum(len(prompts[a]) - min(int(matched[a]), len(prompts[a]) - 1) + max_new[a] for a in adm)
        assert need < lt.rx_evictable_size() + lt.rx_available() or not len(adm)
        assert lt.rx_evictable_size() == ot.evictable_size()
        # run the admitted requests: alloc their new tokens (evict-retry), finish half of them now
        for a in adm:
            n, mm = len(prompts[a]), min(int(matched[a]), len(prompts[a]) - 1)
            s_l = lt.rx_alloc(n - mm)
            if s_l is None:
                lt.rx_evict(n - mm - lt.rx_available())
                ot.evict(n - mm - ot.available())
                s_l = lt.rx_alloc(n - mm)
            s_o = ot.alloc(n - mm)
            assert s_l is not None and list(s_l) == list(s_o)
            pre = list(sl[off[a]:off[a] + mm])
            pinned.append((int(nodes[a]), onodes[a], list(prompts[a]), pre + list(s_l)))
        while pinned and (len(pinned) > 4 or rng.random() < 0.5):
            node, onode, toks, slots = pinned.pop(int(rng.integers(0, len(pinned))))
            assert lt.rx_dec_ref(node) == ot.dec_ref(onode)
            assert lt.rx_insert(toks, slots) == ot.insert(toks, slots)
        assert lt.rx_dump_json() == json.loads(ot.dump_json())


def test_rx_schedule_errors_have_no_side_effect():
    t = LibCache(64)
    t.rx_insert([1, 2, 3], list(t.rx_alloc(3)))
    clock = t.rx_clock() if hasattr(t, "rx_clock") else None
    dump = t.rx_dump_json()
    toks, off = np.array([1, 2, 3, 4], np.int32), np.array([0, 4], np.int64)
    with pytest.raises(RxError):
        t.rx_schedule(toks, off, [1], "random", None)            # RANDOM needs keys
    with pytest.raises(RxError):
        t.rx_schedule(toks, np.array([0, 0], np.int64), [1])     # empty prompt
    with pytest.raises(RxError):
        t.rx_schedule(toks, off, [-1])                           # negative max_new
    assert t.rx_dump_json() == dump
    if clock is not None:
        assert t.rx_clock() == clock
    # empty queue: nothing admitted, nothing touched
    _, _, _, adm, _ = t.rx_schedule(np.zeros(0, np.int32), np.zeros(1, np.int64), [])
    assert len(adm) == 0 and t.rx_dump_json() == dump
