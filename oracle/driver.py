"""Oracle request flow (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

The request flow of Alg. 1, for batches that are admitted
whole (C1/C2/C3/C5: the pool is sized so they fit).  For one batch:

 1. match_prefix every request in list order (Alg. 1 "for req in requests",
    P:526-528); the usable prefix is capped at n-1 (R11) so every request has
    a query row;
 2. increase_ref_counter on every matched node;
 3. alloc(sum of new tokens); on failure evict the shortfall and retry once
    (R6); request i takes the next n_i - m_i slots (R8);
 4. extend attention for all new tokens (B.run);
 5. decode steps: every still-running request allocates one slot per step
    (evict-retry as above), stores its newest token's KV and attends;
 6. a request that produced its last token finishes: decrease_ref_counter
    then insert(prompt + outputs, slots), in batch order.

Generated tokens come from the mock model in rxgen (next_token of the prefix
hash), so both sides see the same token streams.  The KV written to a slot is
identified by the prefix hash of the token it belongs to (rxgen.values); the
oracle's pool stores that hash per slot and expands values on read.

Every tree result is appended to ``trace`` as a plain tuple; slot lists are
kept whole.  tests/ compare this trace with the library's, element by element.
"""
from __future__ import annotations

import numpy as np

from rxgen.hashing import prefix_hashes, next_token, splitmix64_int, MASK64
from rxgen.values import gen_values, KIND_K, KIND_V, KIND_Q

from .radix import RadixCache
from . import attention


class OOM(Exception):
    pass


class Seq:
    """One request while it runs: tokens so far, their hashes, their slots."""

    def __init__(self, rid, prompt, n_out, seed, vocab):
        self.rid = rid
        self.tokens = [int(t) for t in prompt]
        self.hashes = [int(h) for h in prefix_hashes(self.tokens, seed)]
        self.n_prompt = len(self.tokens)
        self.n_out = n_out
        self.vocab = vocab
        self.slots = []
        self.node = None
        self.prefix_len = 0

    def gen_next(self):
        """Mock model: append the token generated after the current last position."""
        h = self.hashes[-1]
        t = next_token(h, self.vocab)
        self.tokens.append(t)
        self.hashes.append(splitmix64_int((h ^ t) & MASK64))


class OracleEngine:
    def __init__(self, wl, sample_extend=None, sample_decode=None, q_scale=1.0, materialize=False, policy="lspf"):
        """sample_extend(call_idx, B, prefix_lens, extend_lens) -> list of (req_idx, j) rows to evaluate, or None (= none);
        sample_decode(call_idx, step, B) -> list of req_idx to evaluate."""
        self.wl = wl
        self.policy = policy        # Alg. 1 queue order ("lspf"; P:432 ablations "fcfs", "random")
        self.shape = wl.shape
        self.tree = RadixCache(wl.num_slots)
        self.slot_hash = {}
        self.trace = []
        self.sample_extend = sample_extend
        self.sample_decode = sample_decode
        self.q_scale = q_scale
        self.extend_calls = 0
        self.decode_calls = 0
        self.outputs = {}           # ("extend", call, req_idx, j) / ("decode", call, req_idx) -> float64 [H_q, hd]
        self.stats = {"prompt_tokens": 0, "cached_prompt_tokens": 0}
        # materialize=True: the pool holds expanded K/V values (written at store time);
        # False: it holds the prefix hash per slot and expands on read (full-size sampled runs)
        self.pool = attention.OraclePool(wl.num_slots, wl.shape.h_kv, wl.shape.head_dim) if materialize else None

    # ------------------------------------------------------------ pool / values
    def _store(self, slots, hashes):
        for s_, h in zip(slots, hashes):
            self.slot_hash[int(s_)] = int(h)
        if self.pool is not None and len(slots):
            hs = np.asarray(hashes, dtype=np.uint64)
            sh = self.shape
            k = gen_values(hs, range(sh.h_kv), KIND_K, sh.head_dim).float().numpy()
            v = gen_values(hs, range(sh.h_kv), KIND_V, sh.head_dim).float().numpy()
            self.pool.store(np.asarray(slots, dtype=np.int64), k, v)

    def _kv(self, slots, g, kind):
        if self.pool is not None:
            arr = self.pool.k if kind == KIND_K else self.pool.v
            return arr[np.asarray(slots, dtype=np.int64), g].astype(np.float64)
        hs = np.array([self.slot_hash[int(s)] for s in slots], dtype=np.uint64)
        return gen_values(hs, [g], kind, self.shape.head_dim)[:, 0].float().numpy().astype(np.float64)

    def _q(self, h, heads):
        return gen_values(np.array([h], dtype=np.uint64), heads, KIND_Q, self.shape.head_dim,
                          scale=self.q_scale)[0].float().numpy().astype(np.float64)

    def _attend(self, seq: Seq, p: int):
        """o[H_q, hd] for the query at absolute position p of seq, read through the pool by slot."""
        sh = self.shape
        G = sh.group
        out = np.zeros((sh.h_q, sh.head_dim))
        slots = seq.slots[:p + 1]
        for g in range(sh.h_kv):
            kmat = self._kv(slots, g, KIND_K)
            vmat = self._kv(slots, g, KIND_V)
            qg = self._q(seq.hashes[p], range(g * G, (g + 1) * G))
            out[g * G:(g + 1) * G] = attention.attend_row(qg, kmat, vmat, sh.sm_scale)
        return out

    # ------------------------------------------------------------ tree steps
    def _alloc(self, n):
        s = self.tree.alloc(n)
        if s is None:
            short = n - self.tree.available()
            evicted, runs = self.tree.evict(short)
            self.trace.append(("evict", short, evicted, tuple(tuple(r) for r in runs)))
            s = self.tree.alloc(n)
            if s is None:
                raise OOM(f"need {n}, available {self.tree.available()}")
        self.trace.append(("alloc", n, tuple(s)))
        return s

    def _finish(self, seq: Seq):
        d = self.tree.dec_ref(seq.node)
        self.trace.append(("dec_ref", seq.rid, d))
        new_cached, dup = self.tree.insert(seq.tokens, seq.slots)
        self.trace.append(("insert", seq.rid, new_cached, dup))

    def _match(self, seqs):
        """Alg. 1 "for req in requests: T.match_prefix"; usable prefix capped at n-1 (R11)."""
        for s in seqs:
            node, m, slots = self.tree.match_prefix(s.tokens[:s.n_prompt])
            self.trace.append(("match", s.rid, m, tuple(slots)))
            s.node = node
            s.matched = m
            s.prefix_len = min(m, s.n_prompt - 1)
            s.slots = list(slots[:s.prefix_len])

    def _seqs(self, reqs):
        return [Seq(r.tag, r.prompt, r.max_new_tokens, self.wl.seed, self.wl.vocab) for r in reqs]

    def run_batch(self, reqs):
        """Run one batch admitted whole: match, pin, then run to completion."""
        seqs = self._seqs(reqs)
        self._match(seqs)
        for s in seqs:
            self.trace.append(("inc_ref", s.rid, self.tree.inc_ref(s.node)))
        return self._run_matched(seqs)

    def run_waves(self, reqs):
        """Alg. 1 admission repeated until every request has run.

        Each wave: match every waiting request, sort the queue by
        self.policy — "lspf": matched length, longest first, ties by arrival
        (P:218); "fcfs": arrival order; "random": ascending rxgen.sched_keys,
        ties by arrival (the ablations of P:432) — then admit while
        req.size() + current < available + delta with available = evictable +
        free updated by the inc_ref delta, delta = the
        candidate's own pin delta (R25), and current += req.size() (R7);
        req.size() = new prompt tokens + max_new_tokens.  The
        admitted batch runs to completion (reading R22: waves instead of
        per-iteration joins)."""
        from rxgen import sched_keys
        waiting = self._seqs(reqs)
        done = []
        wave = 0
        while waiting:
            self._match(waiting)
            idx = list(range(len(waiting)))
            if self.policy == "lspf":
                order = sorted(idx, key=lambda i: (-waiting[i].matched, i))
            elif self.policy == "fcfs":
                order = idx
            elif self.policy == "random":
                keys = [int(k) for k in sched_keys(self.wl.seed, wave, len(waiting))]
                order = sorted(idx, key=lambda i: (keys[i], i))
            else:
                raise ValueError(self.policy)
            available = self.tree.evictable_size() + self.tree.available()
            current = 0
            admitted = []
            for i in order:
                s = waiting[i]
                size = (s.n_prompt - s.prefix_len) + s.n_out
                # reading R25: the fit check counts the candidate's own pin (Alg. 1 checks
                # before pinning, which lets a later pin shrink `available` below what the
                # already-admitted requests need)
                d = self.tree.inc_ref(s.node)
                if size + current < available + d:
                    self.trace.append(("inc_ref", s.rid, d))
                    available += d
                    current += size
                    admitted.append(i)
                else:
                    self.tree.dec_ref(s.node)
            if not admitted:
                raise OOM("no waiting request fits the pool")
            self.trace.append(("admit", tuple(waiting[i].rid for i in admitted)))
            done.extend(self._run_matched([waiting[i] for i in admitted]))
            keep = set(admitted)
            waiting = [s for i, s in enumerate(waiting) if i not in keep]
            wave += 1
        by_rid = {s.rid: s for s in done}
        return [by_rid[r.tag] for r in reqs]

    # ------------------------------------------------------------ constrained decoding (§4)
    def run_fsm_batch(self, reqs):
        """A batch decoding under the workload's regex, admitted whole.

        §4 P:255-266 / App. B, step by step.  The FSM (oracle.fsm, built once for the
        batch) walks with the mock model (rxgen.fsm_choice, R28): at a state the options are
        the allowed bytes, ascending, then STOP if the state is accepting.  Compressed mode: at a
        singular state the whole compressed edge is appended at once (Jump Forward) — from
        the start state it is prefilled with the prompt; after a sampled token it is processed in
        the same forward pass as that token ("decoded in one forward pass").  Normal mode:
        one token per forward pass.  Each forward pass over more than one token of a
        request is an extend call, otherwise a decode call; slots are allocated per pass in batch
        order (R23); a request that chooses STOP finishes (dec_ref + insert) before the next pass."""
        from rxgen import fsm_choice
        from .fsm import FSM
        if getattr(self, "_fsm", None) is None:
            self._fsm = FSM(self.wl.meta["regex"])
        fsm, compressed = self._fsm, self.wl.meta["compressed"]
        seqs = self._seqs(reqs)
        self._match(seqs)
        for s in seqs:
            self.trace.append(("inc_ref", s.rid, self.tree.inc_ref(s.node)))
            self.stats["prompt_tokens"] += s.n_prompt
            self.stats["cached_prompt_tokens"] += s.prefix_len

        def append(s, byte):
            t = byte + 1                              # byte-level vocabulary (R26)
            s.tokens.append(t)
            s.hashes.append(splitmix64_int((s.hashes[-1] ^ t) & MASK64))

        for s in seqs:
            s.state = 0
            if compressed:
                forced, s.state = fsm.jump(0)
                for b in forced:
                    append(s, b)
        # prefill: prompt (beyond the cached prefix) + the start state's forced edge
        ext = [len(s.tokens) - s.prefix_len for s in seqs]
        new = self._alloc(sum(ext))
        off = 0
        for s, n in zip(seqs, ext):
            s.slots.extend(new[off:off + n])
            off += n
        call = self.extend_calls
        self.extend_calls += 1
        self._store([s.slots[p] for s in seqs for p in range(s.prefix_len, len(s.tokens))],
                    [s.hashes[p] for s in seqs for p in range(s.prefix_len, len(s.tokens))])
        for (bi, j) in (self.sample_extend(call, seqs) if self.sample_extend else []):
            if j < ext[bi]:
                self.outputs[("extend", call, bi, j)] = self._attend(seqs[bi], seqs[bi].prefix_len + j)
        running = seqs
        step = 0
        while running:
            # the model's choice after the last processed token of every running request
            still, seg = [], []
            for s in running:
                opts = fsm.allowed(s.state) + (["STOP"] if fsm.accepting[s.state] else [])
                pick = opts[fsm_choice(s.hashes[-1], len(opts))]
                if pick == "STOP":
                    self._finish(s)
                    continue
                start = len(s.tokens)
                append(s, pick)
                s.state = fsm.step(s.state, pick)
                if compressed:
                    forced, s.state = fsm.jump(s.state)
                    for b in forced:
                        append(s, b)
                still.append(s)
                seg.append((start, len(s.tokens) - start))
            running = still
            if not running:
                break
            new = self._alloc(sum(n for _, n in seg))
            off = 0
            for s, (p0, n) in zip(running, seg):
                s.slots.extend(new[off:off + n])
                off += n
            self._store(new, [s.hashes[p] for s, (p0, n) in zip(running, seg) for p in range(p0, p0 + n)])
            if all(n == 1 for _, n in seg):
                call = self.decode_calls
                self.decode_calls += 1
                for bi in (self.sample_decode(call, step, running) if self.sample_decode else []):
                    self.outputs[("decode", call, bi)] = self._attend(running[bi], len(running[bi].tokens) - 1)
            else:
                call = self.extend_calls
                self.extend_calls += 1
                for (bi, j) in (self.sample_extend(call, running) if self.sample_extend else []):
                    if j < seg[bi][1]:
                        self.outputs[("extend", call, bi, j)] = self._attend(running[bi], seg[bi][0] + j)
            step += 1
        self.trace.append(("sizes", self.tree.evictable_size(), self.tree.total_cached(), self.tree.available()))
        return seqs

    def _run_matched(self, seqs):
        for s in seqs:
            self.stats["prompt_tokens"] += s.n_prompt
            self.stats["cached_prompt_tokens"] += s.prefix_len
        # 3. alloc with evict-retry
        ext = [s.n_prompt - s.prefix_len for s in seqs]
        new = self._alloc(sum(ext))
        off = 0
        for s, n in zip(seqs, ext):
            s.slots.extend(new[off:off + n])
            off += n
        # 4. extend: store new KV (slot -> prefix hash), then attend
        call = self.extend_calls
        self.extend_calls += 1
        self._store([s.slots[p] for s in seqs for p in range(s.prefix_len, s.n_prompt)],
                    [s.hashes[p] for s in seqs for p in range(s.prefix_len, s.n_prompt)])
        rows = self.sample_extend(call, seqs) if self.sample_extend else []
        for (bi, j) in rows:
            s = seqs[bi]
            self.outputs[("extend", call, bi, j)] = self._attend(s, s.prefix_len + j)
        # 5./6. finish requests with no outputs, then decode
        for s in seqs:
            if s.n_out == 0:
                self._finish(s)
        running = [s for s in seqs if s.n_out > 0]
        step = 0
        while running:
            for s in running:
                s.gen_next()
            new = self._alloc(len(running))
            for s, slot in zip(running, new):
                s.slots.append(slot)
            self._store(new, [s.hashes[-1] for s in running])
            call = self.decode_calls
            self.decode_calls += 1
            idx = self.sample_decode(call, step, running) if self.sample_decode else []
            for bi in idx:
                s = running[bi]
                self.outputs[("decode", call, bi)] = self._attend(s, len(s.tokens) - 1)
            step += 1
            still = []
            for s in running:
                if len(s.tokens) - s.n_prompt >= s.n_out:
                    self._finish(s)
                else:
                    still.append(s)
            running = still
        self.trace.append(("sizes", self.tree.evictable_size(), self.tree.total_cached(), self.tree.available()))
        return seqs

    # ------------------------------------------------------------ workloads
    def run_workload(self):
        """Run a whole workload (phases for C1/C2/C5; turns for C3)."""
        wl = self.wl
        if wl.name == "C3":
            return self._run_chat()
        if wl.name == "C4":
            return self._run_tot()
        for kind, reqs in wl.phases:
            if kind == "queue":
                self.run_waves(reqs)
            elif kind == "fsm":
                self.run_fsm_batch(reqs)
            else:
                self.run_batch(reqs)
        return self

    def _run_chat(self):
        from rxgen.workloads import Request
        m = self.wl.meta
        hist = [np.asarray(m["system"], dtype=np.int32) for _ in m["turn_inputs"]]
        for t in range(m["turns"]):
            reqs = [Request(np.concatenate([hist[s], m["turn_inputs"][s][t]]), m["turn_outputs"][s][t], f"s{s}t{t}")
                    for s in range(len(hist))]
            done = self.run_batch(reqs)
            hist = [np.asarray(d.tokens, dtype=np.int32) for d in done]
        return self

    def _run_tot(self):
        """C4: tree-of-thought; root as a hint, then each level's branches under Alg. 1 admission."""
        from rxgen.workloads import Request
        m = self.wl.meta
        self.run_batch([Request(np.asarray(m["root"], dtype=np.int32), 0, "root")])
        parents = [np.asarray(m["root"], dtype=np.int32)]
        for lvl, nodes in enumerate(m["levels"]):
            reqs = [Request(np.concatenate([parents[p], bp]), tl, f"L{lvl}n{i}") for i, (p, bp, tl) in enumerate(nodes)]
            parents = [np.asarray(s.tokens, dtype=np.int32) for s in self.run_waves(reqs)]
        return self
