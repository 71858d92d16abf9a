"""Oracle radix tree + token-slot pool (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Follows PAPER.md §3 (lines 176-188) and Alg. 1 (lines 516-569) step by step,
with the readings R1-R10 of SURVEY.md §8(c) / DESIGN.md "Readings":

* the KV pool is paged with one token per page; slot 0 is reserved as
  the padding sink, slots 1..S-1 are allocatable;
* cache and running requests share that one pool;
* alloc(n) returns the n smallest free slots in ascending order (R8);
* a global clock ticks once per match_prefix and once per insert; every node
  on the touched path gets the new value (R1, R9);
* splits happen eagerly, in match_prefix and insert (R3); the upper half is a
  new node (fresh id, copies ref and stamp), the lower half keeps its id,
  stamp and children (R4);
* a node is evictable iff it is a leaf with ref 0; evict removes
  whole leaves in (last_access, id) order (R2, R5) until >= needed tokens;
* insert keeps the tree's slots on already-cached positions and frees the
  caller's differing slots, in position order (R10).

Deliberately plain: a dict of children per node, a sorted Python list of free
slots, a scan-free heap for eviction.  No attempt at speed.
"""
from __future__ import annotations

import bisect
import heapq
import json


class Node:
    __slots__ = ("id", "tokens", "slots", "children", "parent", "ref", "last_access")

    def __init__(self, nid, tokens, slots, parent, ref, last_access):
        self.id = nid
        self.tokens = list(tokens)
        self.slots = list(slots)
        self.children = {}
        self.parent = parent
        self.ref = ref
        self.last_access = last_access


class Underflow(Exception):
    """dec_ref would drive a reference count below zero."""


class RadixCache:
    """One object owns the tree and the slot pool, because they share memory."""

    def __init__(self, num_slots: int):
        assert num_slots >= 1
        self.num_slots = num_slots
        self.free = list(range(1, num_slots))      # sorted ascending
        self.root = Node(0, [], [], None, 0, 0)
        self.next_id = 1
        self.clock = 0

    # ----------------------------------------------------------------- pool
    def available(self) -> int:
        return len(self.free)

    def alloc(self, n: int):
        """n smallest free slots, ascending; None (no side effect) if fewer than n are free."""
        if n < 0:
            raise ValueError("n < 0")
        if n > len(self.free):
            return None
        out = self.free[:n]
        del self.free[:n]
        return out

    def free_slots(self, slots):
        for s in slots:
            if not (1 <= s < self.num_slots):
                raise ValueError(f"slot {s} out of range")
            i = bisect.bisect_left(self.free, s)
            if i < len(self.free) and self.free[i] == s:
                raise ValueError(f"double free of slot {s}")
            self.free.insert(i, s)

    # ----------------------------------------------------------------- tree
    def _split(self, child: Node, k: int) -> Node:
        """Split child's edge after k tokens; return the new upper node (R4)."""
        parent = child.parent
        upper = Node(self.next_id, child.tokens[:k], child.slots[:k], parent, child.ref, child.last_access)
        self.next_id += 1
        parent.children[upper.tokens[0]] = upper
        child.tokens = child.tokens[k:]
        child.slots = child.slots[k:]
        child.parent = upper
        upper.children[child.tokens[0]] = child
        return upper

    @staticmethod
    def _common(a, b) -> int:
        k = 0
        while k < len(a) and k < len(b) and a[k] == b[k]:
            k += 1
        return k

    def match_prefix(self, tokens):
        """Alg. 1 T.match_prefix: (deepest node, matched_len, slots of the matched prefix)."""
        tokens = [int(t) for t in tokens]
        self.clock += 1
        node = self.root
        i = 0
        slots = []
        while i < len(tokens):
            child = node.children.get(tokens[i])
            if child is None:
                break
            k = self._common(child.tokens, tokens[i:])
            if k < len(child.tokens):
                child = self._split(child, k)
            child.last_access = self.clock
            slots.extend(child.slots)
            i += k
            node = child
        return node, i, slots

    def insert(self, tokens, slots):
        """Alg. 1 T.insert: cache tokens with their slots.

        Returns (new_cached, dup_freed).  Ownership of every passed slot moves
        to the cache: slots on already-cached positions that differ from the
        tree's are freed (R10).
        """
        tokens = [int(t) for t in tokens]
        slots = [int(s) for s in slots]
        if len(tokens) != len(slots):
            raise ValueError("tokens/slots length mismatch")
        self.clock += 1
        node = self.root
        i = 0
        dup = []
        while i < len(tokens):
            child = node.children.get(tokens[i])
            if child is None:
                break
            k = self._common(child.tokens, tokens[i:])
            if k < len(child.tokens):
                child = self._split(child, k)
            child.last_access = self.clock
            for j in range(k):
                if slots[i + j] != child.slots[j]:
                    dup.append(slots[i + j])
            i += k
            node = child
        new_cached = len(tokens) - i
        if new_cached:
            leaf = Node(self.next_id, tokens[i:], slots[i:], node, 0, self.clock)
            self.next_id += 1
            node.children[tokens[i]] = leaf
        self.free_slots(dup)
        return new_cached, len(dup)

    def inc_ref(self, node: Node) -> int:
        """Alg. 1 T.increase_ref_counter; returns the change in evictable size (<= 0)."""
        delta = 0
        while node is not self.root:
            if node.ref == 0:
                delta -= len(node.tokens)
            node.ref += 1
            node = node.parent
        return delta

    def dec_ref(self, node: Node) -> int:
        """Alg. 1 T.decrease_ref_counter; returns the change in evictable size (>= 0)."""
        n = node
        while n is not self.root:
            if n.ref < 1:
                raise Underflow(f"node {n.id} ref {n.ref}")
            n = n.parent
        delta = 0
        while node is not self.root:
            node.ref -= 1
            if node.ref == 0:
                delta += len(node.tokens)
            node = node.parent
        return delta

    def _nodes(self):
        out = []
        stack = [self.root]
        while stack:
            n = stack.pop()
            out.append(n)
            stack.extend(n.children.values())
        return out

    def evictable_size(self) -> int:
        return sum(len(n.tokens) for n in self._nodes() if n is not self.root and n.ref == 0)

    def total_cached(self) -> int:
        return sum(len(n.tokens) for n in self._nodes() if n is not self.root)

    def evict(self, needed: int):
        """§3 "evicts the least recently used leaf first"; Alg. 1 T.evict.

        Returns (evicted_tokens, [freed slot runs in eviction order]).
        """
        heap = [(n.last_access, n.id, n) for n in self._nodes()
                if n is not self.root and not n.children and n.ref == 0]
        heapq.heapify(heap)
        evicted = 0
        runs = []
        while evicted < needed and heap:
            _, _, n = heapq.heappop(heap)
            parent = n.parent
            del parent.children[n.tokens[0]]
            n.parent = None
            self.free_slots(n.slots)
            runs.append(list(n.slots))
            evicted += len(n.tokens)
            if parent is not self.root and not parent.children and parent.ref == 0:
                heapq.heappush(heap, (parent.last_access, parent.id, parent))
        return evicted, runs

    # ----------------------------------------------------------------- debug
    def dump(self) -> dict:
        """Deterministic pre-order dump: children ordered by first token."""
        def rec(n):
            return {"id": n.id, "tokens": n.tokens, "slots": n.slots, "ref": n.ref,
                    "last_access": n.last_access,
                    "children": [rec(n.children[t]) for t in sorted(n.children)]}
        return rec(self.root)

    def dump_json(self) -> str:
        return json.dumps(self.dump(), separators=(",", ":"))
