"""The library-side request flow (paper_2312_07104_b200.engine, C++ tree via the
C ABI) against the oracle driver (pure-Python tree): identical tree traces —
every matched length and slot vector, ref delta, allocation, eviction run and
insert result — on the workload shapes C1-C5.  CPU only (plan pass: tree ops,
no kernels)."""
import numpy as np
import pytest

from oracle.driver import OracleEngine
from paper_2312_07104_b200.engine import Engine, shard_heads
from rxgen import workloads


def _traces(wl):
    o = OracleEngine(wl)
    o.run_workload()
    e = Engine(wl, plan_only=True, record=True)
    e.run_workload()
    return o.trace, e.trace


def _cmp(a, b):
    assert len(a) == len(b)
    for i, (x, y) in enumerate(zip(a, b)):
        assert x == y, f"trace entry {i}: oracle {str(x)[:200]} != lib {str(y)[:200]}"


@pytest.mark.parametrize("cfg", [
    lambda: workloads.c1(),
    lambda: workloads.c2(n_req=12, prefix=200, new_lo=5, new_hi=40, decode=6, num_slots=8192),
    lambda: workloads.c3(sessions=10, turns=3, in_lo=5, in_hi=30, out_lo=3, out_hi=12, num_slots=8192),
    lambda: workloads.c5(n_req=8, prefix=300, question=20, decode=5, num_slots=8192),
    lambda: workloads.c4(),
    lambda: workloads.c4(seed=1, root=300, p_lo=8, p_hi=40, t_lo=4, t_hi=20, capacity_frac=0.5),
])
def test_trace_equal(cfg):
    o, e = _traces(cfg())
    _cmp(o, e)


def _evicting_workload(num_slots=700):
    """Four few-shot phases with unrelated prefixes: later phases must evict the
    (ref 0) cache of earlier ones to run (Alg. 1 evict-retry, R6)."""
    from rxgen.workloads import Workload, Request, Shape
    rng = np.random.default_rng(5)
    phases = []
    for ph in range(4):
        pre = rng.integers(1, 30000, 90).astype(np.int32)
        phases.append(("hint", [Request(pre, 0, f"p{ph}")]))
        reqs = [Request(np.concatenate([pre, rng.integers(1, 30000, int(rng.integers(3, 30))).astype(np.int32)]),
                        int(rng.integers(1, 9)), f"p{ph}r{i}") for i in range(6)]
        phases.append(("batch", reqs))
    return Workload("EV", Shape(8, 2, 64), num_slots, 32000, 5, phases)


def test_trace_equal_with_eviction():
    o, e = _traces(_evicting_workload())
    assert sum(t[0] == "evict" for t in o) >= 2
    _cmp(o, e)


def test_hit_rate_few_shot_closed_form():
    """n requests sharing k prefix tokens with q distinct tokens, no hint:
    hit rate (n-1)k / (n(k+q)).  Here the hint is replaced by running requests one per batch."""
    from rxgen.workloads import Request
    rng = np.random.default_rng(0)
    k, q, n = 40, 7, 9
    pre = rng.integers(1, 30000, k).astype(np.int32)
    wl = workloads.c1(n_req=1, prefix=4, new=1, decode=0, num_slots=4096)
    e = Engine(wl, plan_only=True)
    for i in range(n):
        e.run_batch([Request(np.concatenate([pre, rng.integers(1, 30000, q).astype(np.int32)]), 0, f"r{i}")])
    hit = e.stats["cached_prompt_tokens"] / e.stats["prompt_tokens"]
    assert hit == pytest.approx((n - 1) * k / (n * (k + q)))


def test_shard_heads():
    assert shard_heads(64, 8, 0, 8) == (list(range(8)), [0])
    assert shard_heads(64, 8, 1, 2) == (list(range(32, 64)), [4, 5, 6, 7])
    assert shard_heads(8, 2, 3, 4) == ([6, 7], [1])
    assert shard_heads(32, 32, 1, 4) == (list(range(8, 16)), list(range(8, 16)))


def test_c4_admission_waves_and_eviction():
    """C4 at 60% capacity: the deepest level cannot run in one wave (Alg. 1 fit
    check) and finished branches are evicted LRU to make room."""
    o, e = _traces(workloads.c4())
    admits = [t for t in o if t[0] == "admit"]
    assert len(admits) > 3 and sum(t[0] == "evict" for t in o) > 0
    _cmp(o, e)


def test_ragged_flat_matches_loop():
    from paper_2312_07104_b200.engine import _ragged_flat
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(0, 12))
        starts = rng.integers(0, 1000, n)
        lens = rng.integers(0, 9, n)
        ref = np.concatenate([np.arange(s, s + l) for s, l in zip(starts, lens)]) if n else np.zeros(0)
        assert np.array_equal(_ragged_flat(starts, lens), ref.astype(np.int64))


def _decode_evicting_workload(num_slots=420):
    """Earlier phases leave ref-0 cache; a later batch's DECODE steps run the free pool dry, so the
    per-step alloc of rx_decode_steps must evict (R6) mid-phase."""
    from rxgen.workloads import Workload, Request, Shape
    rng = np.random.default_rng(9)
    phases = []
    for ph in range(3):
        pre = rng.integers(1, 30000, 60).astype(np.int32)
        reqs = [Request(np.concatenate([pre, rng.integers(1, 30000, 10).astype(np.int32)]), int(rng.integers(20, 40)),
                        f"p{ph}r{i}") for i in range(4)]
        phases.append(("batch", reqs))
    return Workload("DEV", Shape(8, 2, 64), num_slots, 32000, 9, phases)


def test_decode_steps_evict_mid_phase():
    """rx_decode_steps (Alg. 1's output loop in C++) under memory pressure: evictions happen between
    a phase's decode steps, and the trace equals the oracle's entry for entry."""
    o, e = _traces(_decode_evicting_workload())
    ev_in_decode = [i for i, t in enumerate(o) if t[0] == "evict" and i > 0 and o[i + 1][0] == "alloc"
                    and o[i + 1][1] <= 4]
    assert ev_in_decode, "the workload must evict inside a decode phase"
    _cmp(o, e)


@pytest.mark.parametrize("cfg", [
    lambda: workloads.c3(sessions=10, turns=3, in_lo=5, in_hi=30, out_lo=3, out_hi=12, num_slots=8192),
    lambda: workloads.c4(),
    _decode_evicting_workload,
])
def test_native_decode_loop_equals_python_loop(cfg):
    """The C++ decode-step planner and the Python output loop (still used for jump-forward segments,
    DP workers and the on_decode_plan hook) produce the same trace and the same per-call row hashes."""
    wl = cfg()
    a = Engine(wl, plan_only=True, record=True)
    a.run_workload()
    b = Engine(wl, plan_only=True, record=True)
    b.on_decode_plan = lambda *args: None           # forces the Python loop
    b.run_workload()
    _cmp(a.trace, b.trace)
    assert len(a.calls) == len(b.calls)
    for x, y in zip(a.calls, b.calls):
        assert x.kind == y.kind and np.array_equal(x.hashes, y.hashes)
    assert a.stats["decode_tokens"] == b.stats["decode_tokens"]
