"""Oracle data-parallel router (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md App. A.4: workers keep their own radix trees; the router
keeps a meta-tree ("a trie that tracks all sub-trees and their associated
devices"), dispatches by prefix affinity, and applies worker evictions from a
queue later (weakly consistent).  SPEC S:423-473 gives the interface.

Written plainly as a ONE-TOKEN-PER-NODE trie (no edge compression), each node
holding the set of workers believed to cache that prefix, with reading R24
 for scores and tie-breaks:
  affinity[w] = number of leading tokens whose trie node contains w, stopping
                at the first node without w;
  score[w]    = affinity[w] - load_weight * load[w]; argmax, ties -> smaller
                load -> smaller worker id;
  the chosen worker is credited with the whole request at once (group
  affinity) and its load grows by the request's uncached tokens;
  an eviction clears a worker's mark only where its latest insert is older
  than the eviction (a router clock ticks per insert and per queued eviction),
  so staleness can only over-approximate.
"""
from __future__ import annotations


class _N:
    __slots__ = ("workers", "children", "stamp")

    def __init__(self):
        self.workers = set()
        self.children = {}
        self.stamp = {}          # worker -> router clock of its latest insert through this node


class OracleRouter:
    def __init__(self, num_workers: int):
        self.W = num_workers
        self.root = _N()
        self.queue = []
        self.clock = 0

    def insert(self, w: int, tokens):
        self.clock += 1
        n = self.root
        for t in tokens:
            n = n.children.setdefault(int(t), _N())
            n.workers.add(w)
            n.stamp[w] = self.clock

    def affinity(self, tokens):
        aff = [0] * self.W
        alive = set(range(self.W))
        n = self.root
        for t in tokens:
            n = n.children.get(int(t))
            if n is None:
                break
            alive &= n.workers
            if not alive:
                break
            for w in alive:
                aff[w] += 1
        return aff

    def dispatch(self, requests, loads, load_weight):
        """-> (workers, affinities); loads (list of ints) updated in place."""
        out_w, out_a = [], []
        for toks in requests:
            aff = self.affinity(toks)
            best = min(range(self.W), key=lambda w: (-(aff[w] - load_weight * loads[w]), loads[w], w))
            out_w.append(best)
            out_a.append(aff[best])
            loads[best] += len(toks) - aff[best]
            self.insert(best, toks)
        return out_w, out_a

    def queue_evict(self, w, path, leaf_start):
        self.clock += 1
        self.queue.append((w, [int(t) for t in path], leaf_start, self.clock))

    def sync(self):
        n_applied = 0
        while self.queue:
            w, path, leaf_start, stamp = self.queue.pop(0)
            chain = [self.root]
            n = self.root
            for t in path:
                n = n.children.get(t)
                if n is None:
                    break
                chain.append(n)
            # positions leaf_start .. len(path)-1 are chain[leaf_start+1 ..]
            # only annotations older than the eviction (a later re-insert survives)
            for i in range(leaf_start + 1, len(chain)):
                if chain[i].stamp.get(w, 0) < stamp:
                    chain[i].workers.discard(w)
            # prune childless nodes no worker claims, bottom-up
            for i in range(len(chain) - 1, 0, -1):
                node, parent = chain[i], chain[i - 1]
                if not node.workers and not node.children:
                    del parent.children[path[i - 1]]
                else:
                    break
            n_applied += 1
        return n_applied

    def paths(self):
        """{(worker, token tuple of a maximal claimed path)} — for structural comparisons."""
        out = set()

        def rec(n, pre):
            for t, c in n.children.items():
                p = pre + (t,)
                for w in c.workers:
                    if not any(w in cc.workers for cc in c.children.values()):
                        out.add((w, p))
                rec(c, p)
        rec(self.root, ())
        return out
