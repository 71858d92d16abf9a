"""Data-parallel replicas on the GPU (App. A.4).

A W = 2 ``DPCluster`` whose workers run the real kernels (sequentially on one device — the workers
share nothing on the data path, so one device per worker changes no result) is checked against one
oracle per worker: each oracle replays exactly the request lists its worker ran (frontend hints
included), so its radix-tree trace must equal the worker's bit for bit and every attention row must
be within the north-star tolerance.  Two batches over two few-shot prefixes: the router splits the
first by load, the second by prefix affinity (every request of batch 2 hits its worker's cache)."""
import numpy as np
import pytest
import torch

from oracle.driver import OracleEngine
from rxgen import workloads
from rxgen.workloads import Request

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2312_07104_b200.dp import DPCluster
    from paper_2312_07104_b200.engine import InputBank

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


def _batches(seed=5, groups=2, per_group=8, prefix=300):
    rng = np.random.default_rng(seed)
    pres = [rng.integers(1, 32000, prefix).astype(np.int32) for _ in range(groups)]
    out = []
    for b in range(2):
        reqs = []
        for i in range(groups * per_group):
            g = i % groups
            q = rng.integers(1, 32000, int(rng.integers(16, 60))).astype(np.int32)
            reqs.append(Request(np.concatenate([pres[g], q]), int(rng.integers(2, 6)), f"b{b}r{i}"))
        out.append(reqs)
    return out


def _check_worker(wl, cl, w):
    """Worker w of cluster cl against an oracle that replays exactly its request lists: trace
    bit-exact, every attention row within tolerance.  Returns the number of rows checked."""
    e = cl.workers[w]
    oe = OracleEngine(wl, materialize=True,
                      sample_extend=lambda c, seqs: [(i, j) for i, s in enumerate(seqs)
                                                     for j in range(s.n_prompt - s.prefix_len)],
                      sample_decode=lambda c, st, run: list(range(len(run))))
    for reqs in cl.batches[w]:
        oe.run_batch(reqs)
    assert oe.trace == e.trace, f"worker {w}: radix-tree trace differs from its oracle"
    ext = [x for x in e.outputs if x[0] == "extend"]
    dec = [x for x in e.outputs if x[0] == "decode"]
    errs = []
    for key, ref in oe.outputs.items():
        if key[0] == "extend":
            _, call, bi, j = key
            got = ext[call][1][int(np.sum(ext[call][2]["ext"][:bi])) + j]
        else:
            got = dec[key[1]][1][key[2]]
        errs.append(np.abs(got.float().cpu().double().numpy() - ref).ravel())
    err = np.concatenate(errs)
    assert np.isfinite(err).all()
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (w, err.max(), err.mean())
    return len(errs)


def test_dp_cluster_gpu_vs_per_worker_oracles():
    wl = workloads.c2(n_req=4, prefix=64, decode=2, num_slots=4096)      # shape 32/32/128 + pool only
    batches = _batches()
    W = 2
    plan = DPCluster(wl, W, plan_only=True)
    for reqs in batches:
        plan.run_batch(reqs)
    banks = [InputBank(e.calls, wl.shape, e.heads_q, e.heads_kv, "cuda") for e in plan.workers]
    cl = DPCluster(wl, W, device="cuda", record=True)
    for e in cl.workers:
        e.keep_outputs = True
    for reqs in batches:                             # each worker consumes its own bank across both batches
        cl.run_batch(reqs, banks=banks)
    torch.cuda.synchronize()
    for a, b in zip(plan.assignments, cl.assignments):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    wk2, aff2 = cl.assignments[1]
    assert (aff2 >= 300).all()                       # batch 2: every request lands on its prefix
    assert len(set(wk2.tolist())) == W

    n_rows = sum(_check_worker(wl, cl, w) for w in range(W))
    assert n_rows > 500
    # hit rate: batch 2 reuses every prefix on the worker that holds it
    assert cl.hit_rate() > 0.5


def test_dp_local_worker_with_shadows_gpu():
    """bench.py --parallel dp's per-rank layout on one GPU: worker `local` runs its kernels, the other
    workers are plan-only shadows (host tree replay).  The local worker matches its oracle; every
    worker's trace equals the all-plan cluster's."""
    wl = workloads.c2(n_req=4, prefix=64, decode=2, num_slots=4096)
    batches = _batches(seed=7)
    W = 2
    plan = DPCluster(wl, W, plan_only=True, record=True)
    for reqs in batches:
        plan.run_batch(reqs)
    for local in range(W):
        bank = InputBank(plan.workers[local].calls, wl.shape, plan.workers[local].heads_q,
                         plan.workers[local].heads_kv, "cuda")
        cl = DPCluster(wl, W, device="cuda", record=True, local=local)
        cl.workers[local].keep_outputs = True
        for reqs in batches:
            cl.run_batch(reqs, banks=[bank if w == local else None for w in range(W)])
        torch.cuda.synchronize()
        for w in range(W):
            assert cl.workers[w].trace == plan.workers[w].trace
        assert cl.workers[local].stats["launches"] > 0
        assert _check_worker(wl, cl, local) > 100
