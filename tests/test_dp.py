"""Data-parallel cluster (App. A.4): router + W independent workers.
The paper reports "linear scaling and an optimal cache hit rate" on MMLU with 4
workers; here on the C2 few-shot shape (plan-only workers, CPU): loads
are balanced, each worker prefills the shared prefix once, and a second batch
reuses it on every worker."""
import numpy as np

from paper_2312_07104_b200.dp import DPCluster
from rxgen import workloads


def test_dp_few_shot_balanced_and_near_optimal():
    wl = workloads.c2(n_req=64, prefix=1536, new_lo=64, new_hi=192, decode=4, num_slots=40000)
    reqs = wl.phases[1][1]
    W = 4
    cl = DPCluster(wl, W, plan_only=True, load_weight=1.0)
    cl.run_batch(reqs)
    wk, aff = cl.assignments[0]
    counts = np.bincount(wk, minlength=W)
    assert counts.min() >= 13 and counts.max() <= 19, counts
    # each worker computed the 1536-token prefix exactly once (its hint); every request of
    # the batch then hits it: the optimum for W workers
    cached = sum(e.stats["cached_prompt_tokens"] for e in cl.workers)
    computed = sum(e.stats["prompt_tokens"] - e.stats["cached_prompt_tokens"] for e in cl.workers)
    assert cached == len(reqs) * 1536, cached
    assert computed == W * 1536 + sum(len(r.prompt) - 1536 for r in reqs)
    # batch 2: the prefix is now cached on every worker
    reqs2 = workloads.c2(seed=1, n_req=64, prefix=1536, decode=4).phases[1][1]
    pre = reqs[0].prompt[:1536]
    for r in reqs2:
        r.prompt[:1536] = pre
    before = sum(e.stats["cached_prompt_tokens"] for e in cl.workers)
    cl.run_batch(reqs2)
    after = sum(e.stats["cached_prompt_tokens"] for e in cl.workers)
    # every request hits the prefix; each worker's hint re-matches it (one token recomputed, R11)
    assert after - before == 64 * 1536 + W * 1535
    wk2, aff2 = cl.assignments[1]
    assert (aff2 >= 1536).all()
    assert np.bincount(wk2, minlength=W).min() >= 13


def test_dp_evictions_reach_router():
    """Small worker pools force evictions; the router's queue receives them and, once
    synced, never claims a path a worker no longer holds (quiescent convergence)."""
    rng = np.random.default_rng(3)
    wl = workloads.c1(num_slots=300)
    from rxgen.workloads import Request
    W = 2
    cl = DPCluster(wl, W, plan_only=True, load_weight=1.0, record=True)
    for b in range(6):
        pre = rng.integers(1, 30000, 60).astype(np.int32)
        batch = [Request(np.concatenate([pre, rng.integers(1, 30000, 20).astype(np.int32)]), 3, f"b{b}r{i}")
                 for i in range(4)]
        cl.run_batch(batch)
    assert cl.router.rx_router_queue_len() == 0
    assert any(t[0] == "evict" for e in cl.workers for t in e.trace)     # the pools did evict
    # every router claim is backed by the worker's tree
    for w, e in enumerate(cl.workers):
        dump = e.cache.rx_dump_json()
        stack = [(dump, [])]
        while stack:
            n, pre = stack.pop()
            for c in n["children"]:
                path = pre + c["tokens"]
                aff = cl.router.rx_router_affinity(path)
                _, m, _ = e.cache.rx_match_prefix(path)
                assert aff[w] <= m or aff[w] == len(path)
                stack.append((c, path))


def _dp_workload(W):
    from rxgen.workloads import Request, Workload
    base = workloads.dp_fewshot(workers=W, per_worker=16, q_lo=16, q_hi=48, decode=4)
    m = base.meta
    pres = {}
    for _, reqs in base.phases:
        for r in reqs:
            pres.setdefault(int(r.tag.split("s")[1].split("r")[0]), r.prompt[:m["prefix"]])
    hints = [Request(pres[s].copy(), 0, f"hint{s}") for s in range(m["subjects"])]
    return base, Workload("DP", base.shape, base.num_slots, base.vocab, base.seed,
                          [("dp_batch", hints)] + list(base.phases), m)


def test_dp_weak_scaling_reaches_the_w_worker_optimum():
    """bench.py --parallel dp's workload (App. A.4 P:638 "linear scaling and an optimal cache hit
    rate"): with one hint per subject the router spreads the subjects over the workers by load, then
    sends every question to the worker caching its subject — each prefix is computed once in the
    whole cluster (the W-worker optimum) and per-worker prompt work is balanced for W = 1, 2, 4."""
    for W in (1, 2, 4):
        base, wl = _dp_workload(W)
        cl = DPCluster(wl, W, plan_only=True, load_weight=0.1)
        cl.run_workload()
        st = [e.stats for e in cl.workers]
        prompt = sum(x["prompt_tokens"] for x in st)
        computed = prompt - sum(x["cached_prompt_tokens"] for x in st)
        m = wl.meta
        optimum = m["subjects"] * m["prefix"] + sum(len(r.prompt) - m["prefix"] for _, rq in base.phases for r in rq)
        assert computed == optimum, (W, computed, optimum)
        per = [x["prompt_tokens"] for x in st]
        assert max(per) <= 1.05 * min(per), per


def test_dp_local_shadows_replay_identical_trees():
    """One process per GPU: the local worker runs for real while the others are plan-only shadows;
    every shadow's trace equals that worker's trace in an all-plan cluster (deterministic replay, no
    communication needed for routing)."""
    _, wl = _dp_workload(3)
    ref = DPCluster(wl, 3, plan_only=True, load_weight=0.1, record=True)
    ref.run_workload()
    for local in range(3):
        cl = DPCluster(wl, 3, plan_only=True, load_weight=0.1, record=True, local=local)
        cl.run_workload()
        for w in range(3):
            assert cl.workers[w].trace == ref.workers[w].trace
        for a, b in zip(cl.assignments, ref.assignments):
            assert np.array_equal(a[0], b[0])
