"""Data-parallel RadixAttention (App. A.4).

"each worker maintains its own sub-tree, while the router oversees a meta-tree";
requests are dispatched by prefix affinity; workers commit their evictions to
a queue the router applies "during periods of low activity" (here: at the end
of every batch).  Workers are ordinary ``Engine`` instances (own radix tree,
own KV pool — on their own GPU in a multi-process run, sequentially on one
device or plan-only in tests); the router is librx's C++ ``rx_router``.
"""
from __future__ import annotations

import numpy as np

from . import api
from .engine import Engine


def _common_prefix(seqs) -> int:
    if not seqs:
        return 0
    m = min(len(s) for s in seqs)
    a = np.stack([s[:m] for s in seqs])
    diff = np.nonzero((a != a[0:1]).any(axis=0))[0]
    return int(diff[0]) if len(diff) else m


class DPCluster:
    def __init__(self, wl, workers: int, device="cuda", load_weight: float = 1.0, plan_only=False, record=False,
                 local=None):
        """local=None: every worker runs (plan-only or on `device`, sequentially).  local=w: one
        process per GPU — worker w runs its kernels here; the others are plan-only shadows that
        replay their tree operations on the host, so every rank holds the same router state and
        sees the same eviction reports without communication (the tree ops are deterministic, cf.
        P:235)."""
        self.wl = wl
        self.n = workers
        self.local = local
        self.router = api.Router(workers)
        self.load_weight = load_weight
        self.loads = np.zeros(workers, dtype=np.int64)
        self.workers = []
        for w in range(workers):
            shadow = plan_only or (local is not None and w != local)
            e = Engine(wl, device=device, plan_only=shadow, record=record)
            if local is not None and w != local:
                e.collect_calls = False
            e.evict_listener = (lambda path, leaf_start, w=w: self.router.rx_router_queue_evict(w, path, leaf_start))
            self.workers.append(e)
        self.assignments = []
        self.hint_min = 64
        self.batches = [[] for _ in range(workers)]   # per worker: the request lists it ran, in order

    def run_batch(self, reqs, banks=None):
        """Dispatch one batch (router), run every worker's share (workers are independent: no
        data-path collective), report cached paths, then apply the eviction queue."""
        prompts = [np.asarray(r.prompt, dtype=np.int32) for r in reqs]
        wk, aff = self.router.rx_router_dispatch(prompts, self.loads, self.load_weight)
        self.assignments.append((wk.copy(), aff.copy()))
        done = [None] * len(reqs)
        for w, eng in enumerate(self.workers):
            idx = np.nonzero(wk == w)[0]
            if len(idx) == 0:
                continue
            if banks is not None and banks[w] is not None:
                eng.bank = banks[w]
            sub = [reqs[i] for i in idx]
            # Frontend hint per worker ("the frontend sends the prefix first as a hint"):
            # the share's common prefix is prefilled once on this worker before the share runs
            # (if the worker already holds it, the hint costs one recomputed token, R11).
            lcp = _common_prefix([prompts[i] for i in idx])
            if len(sub) >= 2 and lcp >= self.hint_min:
                from rxgen.workloads import Request
                hint = [Request(prompts[idx[0]][:lcp].copy(), 0, f"hint-w{w}-{len(self.assignments)}")]
                self.batches[w].append(hint)
                h = eng.run_batch(hint)[0]
                self.router.rx_router_insert(w, h.tokens[:h.n_prompt])
            self.batches[w].append(sub)
            out = eng.run_batch(sub)
            for i, r in zip(idx, out):
                done[i] = r
                # the worker cached prompt + generated tokens: tell the router about the whole sequence
                self.router.rx_router_insert(w, r.tokens[:r.n_prompt + r.n_out])
        self.loads[:] = 0                      # the batch ran to completion
        self.router.rx_router_sync()
        return done

    def reset(self):
        """Fresh router, trees and pools for another pass (device pools and input banks are kept)."""
        self.router = api.Router(self.n)
        self.loads[:] = 0
        self.assignments = []
        self.batches = [[] for _ in range(self.n)]
        for e in self.workers:
            e.reset()

    def run_workload(self, banks=None):
        for kind, reqs in self.wl.phases:
            assert kind == "dp_batch", kind
            self.run_batch(reqs, banks)
        return self

    def hit_rate(self):
        p = sum(e.stats["prompt_tokens"] for e in self.workers)
        c = sum(e.stats["cached_prompt_tokens"] for e in self.workers)
        return c / max(1, p)
