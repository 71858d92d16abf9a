"""Pins for the oracle's Alg. 1 admission, ``OracleEngine.run_waves`` (oracle/driver.py), against
results the paper and the mathematics fix — not against a restatement of its own formula.

* Theorem 1 (§3, proof P:578-618): for a batch whose radix tree T has edges e,
  every order computes at least C = sum_e |e| prefill tokens, and the longest-shared-prefix-first
  (LSPF) order with a cache >= the longest request computes exactly C.  The test drives the
  oracle's own admission loop (match the queue, sort, fit check, pin, run, finish, insert) and reads
  the computed tokens from its stats; C is counted independently (distinct non-empty prefixes),
  and a brute force over every permutation on a separate plain prefix-set model confirms that no
  order does better.  Request tails are long enough that the Alg. 1 fit check admits one
  request per wave, so the sequential setting of the theorem is what run_waves executes.
* SPEC S:231 few-shot closed form: n requests sharing k tokens with distinct q-token suffixes,
  one at a time, hit rate (n-1)k / (n(k+q)).
* The ablation claim ("cache thrashing", P:432 FCFS / random bars) on the ORACLE's stats:
  on an interleaved multi-prefix queue LSPF > random > FCFS, FCFS = 0.
"""
import itertools
import random

import numpy as np
import pytest

from oracle.driver import OracleEngine
from rxgen import workloads
from rxgen.workloads import Request, Shape, Workload


def _distinct_prefixes(reqs):
    """|edges(T)| summed = number of distinct non-empty prefixes of the request set."""
    return len({tuple(r[:i]) for r in reqs for i in range(1, len(r) + 1)})


def _computed_in_order(reqs, order):
    """Prefill tokens computed when requests run one by one in `order` with an unbounded cache:
    a plain set of cached prefixes (no radix tree, no eviction — capacity is never binding when it
    is >= the longest request and the order is DFS, and with unbounded capacity no order can do
    better than the bound either)."""
    cached = set()
    total = 0
    for i in order:
        r = reqs[i]
        m = max((k for k in range(len(r) + 1) if tuple(r[:k]) in cached or k == 0), default=0)
        total += len(r) - m
        cached.update(tuple(r[:k]) for k in range(1, len(r) + 1))
    return total


def _tree_batch(rng, n_req, tail):
    """Random request tree over a 5-token alphabet; every request ends in a private tail of `tail`
    tokens drawn from a disjoint alphabet, so no request is a prefix of another."""
    stems = []
    while len(stems) < n_req:
        base = stems[rng.randrange(len(stems))] if stems and rng.random() < 0.7 else []
        cut = rng.randrange(0, len(base) + 1) if base else 0
        stems.append(base[:cut] + [rng.randrange(1, 6) for _ in range(rng.randrange(1, 5))])
    return [s + [1000 + 100 * i + j for j in range(tail)] for i, s in enumerate(stems)]


def _queue_workload(reqs, num_slots, name="TH1"):
    return Workload(name, Shape(8, 2, 64), num_slots, 32000, 0,
                    [("queue", [Request(np.asarray(r, np.int32), 0, f"r{i}") for i, r in enumerate(reqs)])])


@pytest.mark.parametrize("seed", range(16))
def test_theorem1_through_run_waves(seed):
    rng = random.Random(seed)
    n = rng.randrange(3, 7)
    stem_max = 4 * n                                  # stems grow by <= 4 tokens per request
    tail = stem_max + 2                               # 2 * tail >= capacity - 1: one admission per wave
    reqs = _tree_batch(rng, n, tail)
    cap = max(len(r) for r in reqs) + 2               # >= longest request (+ padding slot, strict `<` P:540)
    assert 2 * tail >= cap - 1
    o = OracleEngine(_queue_workload(reqs, cap), policy="lspf")
    o.run_workload()
    admits = [t for t in o.trace if t[0] == "admit"]
    assert len(admits) == n and all(len(a[1]) == 1 for a in admits)     # sequential, as in the theorem
    computed = o.stats["prompt_tokens"] - o.stats["cached_prompt_tokens"]
    C = _distinct_prefixes(reqs)
    assert computed == C                                                  # C = sum |e|
    assert min(_computed_in_order(reqs, p) for p in itertools.permutations(range(n))) == C
    total = sum(len(r) for r in reqs)
    assert o.stats["cached_prompt_tokens"] / o.stats["prompt_tokens"] == pytest.approx(1 - C / total)


def test_theorem1_bound_holds_for_every_policy_and_fcfs_can_miss_it():
    """The lower bound C <= computed holds for FCFS and random orders through run_waves too,
    and on some request trees FCFS computes strictly more than C (the order matters)."""
    worse = 0
    for seed in range(30):
        rng = random.Random(500 + seed)
        n = rng.randrange(4, 7)
        tail = 4 * n + 2
        reqs = _tree_batch(rng, n, tail)
        cap = max(len(r) for r in reqs) + 2
        C = _distinct_prefixes(reqs)
        for pol in ("fcfs", "random"):
            o = OracleEngine(_queue_workload(reqs, cap), policy=pol)
            o.run_workload()
            computed = o.stats["prompt_tokens"] - o.stats["cached_prompt_tokens"]
            assert computed >= C
            worse += pol == "fcfs" and computed > C
    assert worse > 0


@pytest.mark.parametrize("n,k,q", [(9, 40, 47), (5, 100, 120), (12, 16, 30)])
def test_few_shot_closed_form_through_run_waves(n, k, q):
    """(n-1)k / (n(k+q)).  The pool (k + q + 2 slots) admits one request per wave (2q > k + q
    + 1 - k), so each request after the first finds the k shared tokens cached."""
    rng = np.random.default_rng(n * 1000 + k)
    pre = rng.integers(1, 30000, k)
    reqs = [list(pre) + list(rng.integers(30000, 60000, q)) for _ in range(n)]
    o = OracleEngine(_queue_workload(reqs, k + q + 2, "FS"), policy="lspf")
    o.run_workload()
    assert all(len(t[1]) == 1 for t in o.trace if t[0] == "admit")
    hit = o.stats["cached_prompt_tokens"] / o.stats["prompt_tokens"]
    assert hit == pytest.approx((n - 1) * k / (n * (k + q)))


def test_few_shot_one_wave_without_hint_has_no_hits():
    """With a pool that admits the whole queue in one wave and no hint, every request is
    matched before any runs: hit rate 0 (why the frontend hint exists)."""
    rng = np.random.default_rng(1)
    pre = rng.integers(1, 30000, 50)
    reqs = [list(pre) + list(rng.integers(30000, 60000, 10)) for _ in range(6)]
    o = OracleEngine(_queue_workload(reqs, 4096, "FS1"), policy="lspf")
    o.run_workload()
    assert len([t for t in o.trace if t[0] == "admit"]) == 1
    assert o.stats["cached_prompt_tokens"] == 0


def test_ablation_on_oracle_stats():
    """P:214-216 / P:432: LSPF > random > FCFS on the MIX queue, FCFS thrashes to 0 — measured on
    the oracle's own run_waves (the library's scheduler is compared to it in test_scheduler.py)."""
    wl = workloads.mix()
    hits = {}
    for p in ("lspf", "fcfs", "random"):
        o = OracleEngine(wl, policy=p)
        o.run_workload()
        hits[p] = o.stats["cached_prompt_tokens"] / o.stats["prompt_tokens"]
    assert hits["lspf"] > hits["random"] > hits["fcfs"]
    assert hits["fcfs"] == 0.0
    assert hits["lspf"] > 0.85


def test_waves_fit_check_never_overcommits():
    """Reading R25: after every admission the admitted sizes fit evictable + free, so the wave's
    allocation (evict-retry) never fails — on C4 at 60 % capacity and on MIX."""
    for wl in (workloads.c4(), workloads.mix()):
        o = OracleEngine(wl)
        o.run_workload()                      # raises OOM on an overcommitted wave
        assert any(t[0] == "admit" for t in o.trace)


def test_fit_check_is_strict_as_in_alg1():
    """Alg. 1 admits iff req.size() + current_size < available_size (strict): a request that
    needs exactly every allocatable slot is not admitted; one more slot and it is."""
    from oracle.driver import OOM
    n = 30
    reqs = [list(range(1, n + 1))]
    with pytest.raises(OOM):
        OracleEngine(_queue_workload(reqs, n + 1)).run_workload()      # n allocatable (slot 0 reserved)
    o = OracleEngine(_queue_workload(reqs, n + 2))
    o.run_workload()
    assert [t for t in o.trace if t[0] == "admit"] == [("admit", ("r0",))]
