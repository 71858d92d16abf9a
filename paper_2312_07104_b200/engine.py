"""Request-flow harness over librx (SURVEY §3 "Build, planned"; L4 in SURVEY §1).

Drives one workload (rxgen.workloads C1-C5) through the paper's flow — Alg. 1
 for batches admitted whole — calling only the C ABI:

  match_prefix -> inc_ref -> alloc (evict shortfall, retry once) ->
  rx_extend (store new KV + attend) -> decode steps (alloc 1 slot/request,
  rx_store_kv + rtt append, rx_decode) -> dec_ref -> insert.

Usable prefix is capped at n-1 so every request has a query row (R11).

Two passes:
  * plan pass (``plan_only=True``): tree ops only; records, per attention
    call, the prefix hashes of the rows it will process;
  * execute pass: same tree ops (deterministic, so identical results) plus the
    kernels, with inputs taken from an ``InputBank`` generated from the plan
    BEFORE any timing (inputs resident in HBM when timing starts).

Tensor parallelism (§3, "each GPU maintains a sharded KV cache.
There is no need for additional synchronization because the tree operations
are the same"): rank r of P owns q heads [r*H_q/P, (r+1)*H_q/P) and the kv
heads they read; every rank runs the identical tree ops; outputs are
reassembled by one all_gather per attention call (see ``tp.py``).
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from rxgen.hashing import prefix_hashes, next_token, splitmix64_int, MASK64
from rxgen.values import gen_values, gen_values_np, KIND_K, KIND_V, KIND_Q

from . import api


def _ragged_flat(starts, lens):
    """concat(arange(s, s + n) for s, n in zip(starts, lens)) without a Python loop."""
    lens = np.asarray(lens, dtype=np.int64)
    total = int(lens.sum())
    excl = np.cumsum(lens) - lens
    return np.repeat(np.asarray(starts, dtype=np.int64) - excl, lens) + np.arange(total, dtype=np.int64)


class OutOfSlots(RuntimeError):
    pass


# RX_CASCADE_STABLE=0: cascade decode steps without a stable region (A/B knob)
_NO_CAS_STABLE = os.environ.get("RX_CASCADE_STABLE", "1") == "0"
# RX_DECODE_PER_STEP=1: one Python-level library call per decode step instead of rx_decode_run (A/B)
_PER_STEP_LAUNCH = os.environ.get("RX_DECODE_PER_STEP", "0") == "1"


def shard_heads(h_q: int, h_kv: int, rank: int, size: int):
    """(q heads, kv heads) owned by this TP rank; kv heads replicated when size > h_kv."""
    assert h_q % size == 0, "h_q must divide by the TP size"
    qh = list(range(rank * h_q // size, (rank + 1) * h_q // size))
    G = h_q // h_kv
    kvh = sorted({h // G for h in qh})
    return qh, kvh


class _Req:
    __slots__ = ("rid", "tokens", "hashes", "n_prompt", "n_out", "node", "prefix", "slots", "row", "matched",
                 "first", "segs")

    def __init__(self, rid, prompt, n_out, seed, vocab, full=None, first=0, segs=None):
        self.rid = rid
        self.n_prompt = len(prompt)
        self.n_out = n_out
        # output schedule: `first` output tokens ride along with the prompt's extend (a jump-forward
        # edge at the FSM start), then one forward pass per segment of segs[k] tokens (1 = a decode
        # step; > 1 = a sampled token plus its jump-forward edge, an extend step)
        self.first = first
        self.segs = np.ones(n_out - first, dtype=np.int64) if segs is None else np.asarray(segs, dtype=np.int64)
        if full is None:
            toks = [int(t) for t in prompt]
            hs = [int(h) for h in prefix_hashes(toks, seed)]
            for _ in range(n_out):
                h = hs[-1]
                t = next_token(h, vocab)
                toks.append(t)
                hs.append(splitmix64_int((h ^ t) & MASK64))
            # arrays, so every C-ABI call passes a pointer without conversion
            full = (np.asarray(toks, dtype=np.int32), np.asarray(hs, dtype=np.uint64))
        self.tokens, self.hashes = full
        self.node = 0
        self.prefix = 0
        self.slots = None
        self.row = 0


@dataclass
class CallPlan:
    kind: str                       # "extend" | "decode"
    hashes: np.ndarray              # uint64 hashes of the rows (query tokens) of the call, packed
    meta: dict = field(default_factory=dict)


class InputBank:
    """q / k / v of every attention call of a workload, on the device, packed per call."""

    def __init__(self, calls, shape, heads_q, heads_kv, device, q_scale=1.0, host=False):
        """host=True: values are generated on the host (rxgen.gen_values_np) into one pinned buffer
        and moved with ONE host-to-device copy (no generator kernels on the device: smoke() uses this
        so a launch list of the run shows only the rx kernels)."""
        self.ext = []
        self.dec = []
        hd = shape.head_dim
        if host:
            parts = []
            for c in calls:
                h = np.asarray(c.hashes, dtype=np.uint64)
                parts.append([gen_values_np(h, heads_q, KIND_Q, hd, scale=q_scale),
                              gen_values_np(h, heads_kv, KIND_K, hd), gen_values_np(h, heads_kv, KIND_V, hd)])
            flat = np.concatenate([a.ravel() for tr in parts for a in tr]) if parts else np.zeros(0, np.float32)
            buf = torch.from_numpy(flat).to(torch.bfloat16).pin_memory().to(device, non_blocking=False)
            off = 0
            for c, tr in zip(calls, parts):
                views = []
                for a in tr:
                    views.append(buf[off:off + a.size].view(a.shape))
                    off += a.size
                (self.ext if c.kind == "extend" else self.dec).append(tuple(views))
            return
        for c in calls:
            h = c.hashes
            q = gen_values(h, heads_q, KIND_Q, hd, scale=q_scale, device=device)
            k = gen_values(h, heads_kv, KIND_K, hd, device=device)
            v = gen_values(h, heads_kv, KIND_V, hd, device=device)
            (self.ext if c.kind == "extend" else self.dec).append((q, k, v))

    def nbytes(self):
        return sum(t.numel() * t.element_size() for lst in (self.ext, self.dec) for tr in lst for t in tr)


class Engine:
    def __init__(self, wl, device="cuda", tp_rank=0, tp_size=1, plan_only=False, record=False,
                 keep_outputs=False, gather=None, cascade=True, policy="lspf"):
        self.wl = wl
        self.policy = policy                  # Alg. 1 queue order: "lspf" (paper), "fcfs", "random"
        self.shape = wl.shape
        self.device = device
        self.plan_only = plan_only
        self.collect_calls = True             # plan pass: record per-call row hashes (input generation)
        self.record = record
        self.keep_outputs = keep_outputs
        self.gather = gather                  # callable(local o) -> full o, or None (P == 1)
        self.heads_q, self.heads_kv = shard_heads(wl.shape.h_q, wl.shape.h_kv, tp_rank, tp_size)
        self.hq, self.hkv = len(self.heads_q), len(self.heads_kv)
        self.cfg = api.attn_cfg(self.hq, self.hkv, wl.shape.head_dim, wl.shape.sm_scale)
        self.cache = api.RadixCache(wl.num_slots)
        self.trace = []
        self.calls = []                      # CallPlan per attention call (plan pass)
        self.outputs = []                    # (kind, o tensor, meta) per call if keep_outputs
        self.stats = {"prompt_tokens": 0, "cached_prompt_tokens": 0, "extend_tokens": 0, "decode_tokens": 0,
                      "output_tokens": 0, "tree_s": 0.0, "launches": 0}
        self._ext_i = 0
        self._dec_i = 0
        self.bank = None
        self._full_cache = {}
        self.timer = None
        self._pin_cache = {}                 # name -> pinned buffer checked out
        self._pin_pool = []                   # (pinned buffer, event of its last H2D copy)
        self.sink = None                     # callable(kind, o) invoked after every attention call
        self.evict_listener = None           # callable(path tokens, leaf_start) per evicted leaf (DP workers)
        # shared-prefix (cascade) decode when the batch shares >= cascade_min_len cached slots
        self.cascade = cascade
        self.cascade_min_len = 256
        # G = 1 (no GQA grouping): below 8 requests the per-request decode (one fused launch + merge)
        # beats the 3-launch cascade chain (2k shared, B = 4: 27.0 vs 33.2 us per step; B = 16:
        # 52.3 vs 32.5 — profiles/r2_cascade_c4_threshold.txt)
        self.cascade_min_batch = 8 if wl.shape.h_q == wl.shape.h_kv else 4
        self._shared = 0
        self._match_cache = {}               # batch key -> (concatenated prompts, offsets)
        self._match_out = None               # reused slot output buffer of _match
        self._slot_bufs = []                 # reused host req_to_token mirrors, one per batch of a pass
        self._slot_buf_i = 0
        self._ws = None
        self._rtt = None
        self._fsm = None                      # compressed FSM of the workload's regex (JSON workload)
        self.on_decode_plan = None            # callable(engine, slots, running, pos) per planned decode step
        self.launch_chunk = int(os.environ.get("RX_LAUNCH_CHUNK", "32"))   # output steps planned per launch batch
        self.gather_chunk_rows = 8192         # TP: extend rows per overlapped all-gather block
        self._ring = 0                        # rotating pinned staging buffers for decode metadata
        self._ext_ring = 0                    # ... and for extend metadata + tables
        if not plan_only:
            hd = wl.shape.head_dim
            self.k_pool = torch.zeros((wl.num_slots, self.hkv, hd), dtype=torch.bfloat16, device=device)
            self.v_pool = torch.zeros_like(self.k_pool)

    # ------------------------------------------------------------------ tree helpers
    def _rec(self, *t):
        if self.record:
            self.trace.append(t)

    def _alloc(self, n):
        c = self.cache
        s = c.rx_alloc(n)
        if s is None:
            short = n - c.rx_available()
            if self.evict_listener is not None:
                # data-parallel worker: report evicted token paths to the router's queue (App. A.4)
                ev, paths = c.rx_evict_paths(short)
                runs = [sl for _, _, sl in paths]
                for path, leaf_start, _ in paths:
                    self.evict_listener(path, leaf_start)
            else:
                ev, runs = c.rx_evict(short)
            self._rec("evict", short, ev, tuple(tuple(int(x) for x in r) for r in runs))
            s = c.rx_alloc(n)
            if s is None:
                raise OutOfSlots(f"need {n}, available {c.rx_available()}")
        if self.record:
            self._rec("alloc", n, tuple(int(x) for x in s))
        return s

    # ------------------------------------------------------------------ one batch
    def _reqs(self, reqs):
        wl = self.wl
        rs = []
        for q in reqs:
            key = (q.tag, len(q.prompt), q.max_new_tokens)
            r = _Req(q.tag, q.prompt, q.max_new_tokens, wl.seed, wl.vocab, self._full_cache.get(key))
            self._full_cache[key] = (r.tokens, r.hashes)
            rs.append(r)
        return rs

    def _fsm_reqs(self, reqs):
        """Requests decoding under the workload's regex (§4): the output is the mock
        model's walk of the compressed FSM (library rx_fsm_*, built once and reused for the batch,
        P:442); compressed mode groups each sampled token with the jump-forward edge that follows
        it, so one forward pass covers the whole segment."""
        from rxgen import fsm_choice
        wl = self.wl
        if self._fsm is None:
            self._fsm = api.Fsm(wl.meta["regex"])
        fsm, compressed = self._fsm, wl.meta["compressed"]
        rs = []
        for q in reqs:
            key = ("fsm", q.tag, len(q.prompt), compressed)
            if key in self._full_cache:
                toks, hs, first, segs = self._full_cache[key]
            else:
                toks = [int(t) for t in q.prompt]
                hs = [int(h) for h in prefix_hashes(toks, wl.seed)]

                def emit(byte):
                    t = byte + 1                      # byte-level vocabulary (R26)
                    hs.append(splitmix64_int((hs[-1] ^ t) & MASK64))
                    toks.append(t)
                st, first, segs = 0, 0, []
                if compressed:
                    forced, st = fsm.rx_fsm_jump(0)
                    for b in forced:
                        emit(b)
                    first = len(forced)
                while True:
                    opts = fsm.rx_fsm_allowed(st) + ([-1] if fsm.rx_fsm_is_accepting(st) else [])
                    pick = opts[fsm_choice(hs[-1], len(opts))]
                    if pick < 0:                      # STOP
                        break
                    emit(pick)
                    st = fsm.rx_fsm_step(st, pick)
                    n = 1
                    if compressed:
                        forced, st = fsm.rx_fsm_jump(st)
                        for b in forced:
                            emit(b)
                        n += len(forced)
                    segs.append(n)
                toks = np.asarray(toks, dtype=np.int32)
                hs = np.asarray(hs, dtype=np.uint64)
                self._full_cache[key] = (toks, hs, first, segs)
            rs.append(_Req(q.tag, q.prompt, len(toks) - len(q.prompt), wl.seed, wl.vocab, (toks, hs), first, segs))
        return rs

    def run_fsm_batch(self, reqs):
        """One batch of regex-constrained requests admitted whole (as run_batch)."""
        t0 = time.perf_counter()
        rs = self._fsm_reqs(reqs)
        self._match(rs)
        deltas = self.cache.rx_inc_ref_batch([r.node for r in rs])
        for r, d in zip(rs, deltas):
            self._rec("inc_ref", r.rid, int(d))
        self.stats["tree_s"] += time.perf_counter() - t0
        return self._run_matched(rs)

    def _match(self, rs):
        """match_prefix for every request (Alg. 1); usable prefix capped at n-1 (R11)."""
        c = self.cache
        if not rs:
            return
        # the batch's concatenated prompts are the same every pass (cached by request identity), and
        # the slot output goes into a reused buffer: fresh multi-MB arrays per batch cost page faults
        key = tuple((r.rid, r.n_prompt) for r in rs)
        hit = self._match_cache.get(key)
        if hit is None:
            toks = np.concatenate([r.tokens[:r.n_prompt] for r in rs])
            off = np.zeros(len(rs) + 1, dtype=np.int64)
            off[1:] = np.cumsum([r.n_prompt for r in rs])
            hit = self._match_cache[key] = (toks, off)
        toks, off = hit
        if self._match_out is None or len(self._match_out) < len(toks):
            self._match_out = np.empty(max(len(toks), 1), dtype=np.int32)
        nodes, matched, sl = c.rx_match_prefix_batch(toks, off, out=self._match_out)   # one C call
        for b, r in enumerate(rs):
            m = int(matched[b])
            s = sl[off[b]:off[b] + m]          # (a view of the reused buffer: valid until the next match)
            if self.record:
                self._rec("match", r.rid, m, tuple(int(x) for x in s))
            r.node = int(nodes[b])
            r.matched = m
            r.prefix = min(m, r.n_prompt - 1)
            r.slots = s[:r.prefix]

    def run_batch(self, reqs):
        """One batch admitted whole: match, pin every request, run to completion."""
        t0 = time.perf_counter()
        rs = self._reqs(reqs)
        self._match(rs)
        deltas = self.cache.rx_inc_ref_batch([r.node for r in rs])
        for r, d in zip(rs, deltas):
            self._rec("inc_ref", r.rid, int(d))
        self.stats["tree_s"] += time.perf_counter() - t0
        return self._run_matched(rs)

    def run_waves(self, reqs):
        """Alg. 1 admission (R7) repeated until every request ran (waves, R22).

        One rx_schedule call per wave (library C++): match every waiting request, order the queue by
        self.policy (LSPF = longest matched prefix first, ties by arrival; FCFS; RANDOM with keys
        from rxgen.sched_keys), admit while size + current < available, available = evictable +
        free updated by the inc_ref delta, current += size, size = new prompt tokens + max_new."""
        from rxgen import sched_keys
        c = self.cache
        waiting = self._reqs(reqs)
        done = {}
        wave = 0
        while waiting:
            t0 = time.perf_counter()
            toks = np.concatenate([r.tokens[:r.n_prompt] for r in waiting])
            off = np.zeros(len(waiting) + 1, dtype=np.int64)
            off[1:] = np.cumsum([r.n_prompt for r in waiting])
            keys = sched_keys(self.wl.seed, wave, len(waiting)) if self.policy == "random" else None
            nodes, matched, sl, adm, deltas = c.rx_schedule(toks, off, [r.n_out for r in waiting], self.policy, keys)
            for b, r in enumerate(waiting):
                m = int(matched[b])
                if self.record:
                    self._rec("match", r.rid, m, tuple(int(x) for x in sl[off[b]:off[b] + m]))
                r.node = int(nodes[b])
                r.matched = m
                r.prefix = min(m, r.n_prompt - 1)
                r.slots = sl[off[b]:off[b] + r.prefix]
            admitted = [int(i) for i in adm]
            for i, d in zip(admitted, deltas):
                self._rec("inc_ref", waiting[i].rid, int(d))
            if not admitted:
                raise OutOfSlots("no waiting request fits the pool")
            self._rec("admit", tuple(waiting[i].rid for i in admitted))
            self.stats["tree_s"] += time.perf_counter() - t0
            for r in self._run_matched([waiting[i] for i in admitted]):
                done[r.rid] = r
            keep = set(admitted)
            waiting = [r for i, r in enumerate(waiting) if i not in keep]
            wave += 1
        return [done[q.tag] for q in reqs]

    def _run_matched(self, rs):
        t0 = time.perf_counter()
        B = len(rs)
        c = self.cache
        n_prompt = np.array([r.n_prompt for r in rs], dtype=np.int64)
        n_out = np.array([r.n_out for r in rs], dtype=np.int64)
        first = np.array([r.first for r in rs], dtype=np.int64)
        stride = int((n_prompt + n_out).max())
        slots = self._slot_buf(B, stride, zero=False)        # host mirror of this batch's req_to_token rows
        prefix = np.array([r.prefix for r in rs], dtype=np.int64)
        for b, r in enumerate(rs):
            slots[b, :r.prefix] = r.slots
        self.stats["prompt_tokens"] += int(n_prompt.sum())
        self.stats["cached_prompt_tokens"] += int(prefix.sum())
        self.stats["output_tokens"] += int(n_out.sum())
        ext = n_prompt + first - prefix
        new = self._alloc(int(ext.sum()))
        off = 0
        for b in range(B):
            e = prefix[b] + ext[b]
            slots[b, prefix[b]:e] = new[off:off + ext[b]]
            slots[b, e:] = 0                                   # positions the output steps fill later
            off += ext[b]
        self.stats["tree_s"] += time.perf_counter() - t0
        self._slots_host = slots
        # cached prefix shared by every request of the batch (same radix path => same slots):
        # decode steps attend it once for the whole batch (rx_decode_cascade_append)
        mp = int(prefix.min())
        if self.cascade and B >= self.cascade_min_batch and mp >= self.cascade_min_len:
            if (slots[:, 0] != slots[0, 0]).any():
                self._shared = 0             # rows differ at position 0: nothing shared (e.g. C3 sessions)
            elif all(r.node == rs[0].node for r in rs):
                self._shared = mp            # one matched radix node: identical slots up to its depth
            else:
                diff = np.nonzero((slots[:, :mp] != slots[0:1, :mp]).any(axis=0))[0]
                self._shared = int(diff[0]) if len(diff) else mp
        else:
            self._shared = 0
        if self._shared < self.cascade_min_len:
            self._shared = 0
        self._extend(rs, slots, prefix, ext)
        # positions every later decode step may read before its programmatic-dependency wait:
        # those written by this batch's prefill (plain launches, complete before the first step)
        self._stable = (n_prompt + first).astype(np.int32)
        t0 = time.perf_counter()
        nseg = np.array([len(r.segs) for r in rs], dtype=np.int64)
        self._finish_many(rs, np.nonzero(nseg == 0)[0], slots)
        running = np.nonzero(nseg > 0)[0]
        self.stats["tree_s"] += time.perf_counter() - t0
        # Output phase, host ahead of the device: the tree ops of each step — its slots (R23: per
        # step, in batch order), finished requests' dec_ref + insert — need no GPU result (the
        # mock-model tokens are known), so steps are planned in chunks and each chunk is launched
        # while the host plans the next.
        cur = n_prompt + first
        unit = all(r.first == 0 and (len(r.segs) == 0 or int(r.segs.max()) == 1) for r in rs)
        if unit and self.on_decode_plan is None and self.evict_listener is None:
            # Alg. 1's output loop in the library: one C call plans launch_chunk iterations (allocs,
            # table rows, device staging records, finishes) — no per-step Python
            self._decode_loop_native(rs, slots, cur, running, n_prompt + n_out)
        else:
            self._output_loop_py(rs, slots, cur, running, nseg, unit)
        self._rec("sizes", c.rx_evictable_size(), c.rx_total_cached(), c.rx_available())
        return rs

    def _slot_buf(self, B, stride, zero=True):
        """A zeroed [B, stride] int32 host mirror for the pass's next batch: buffers are reused
        across passes (k-th batch of a pass -> k-th buffer; a pass keeps every batch's mirror alive
        for its decode_bytes records), so steady state writes warm pages instead of faulting fresh
        ones."""
        i = self._slot_buf_i
        self._slot_buf_i += 1
        if i == len(self._slot_bufs):
            self._slot_bufs.append(np.zeros(0, dtype=np.int32))
        if self._slot_bufs[i].size < B * stride:
            self._slot_bufs[i] = np.zeros(B * stride, dtype=np.int32)
        out = self._slot_bufs[i][:B * stride].reshape(B, stride)
        if zero:
            out.fill(0)
        return out

    def _decode_loop_native(self, rs, slots, cur, running, end):
        """Plain decoding through rx_decode_steps: each C call plans launch_chunk iterations of
        Alg. 1's output loop (alloc + evict-retry, table rows, finishes) and writes their device
        staging records straight into a pinned buffer, which one H2D moves before the chunk's
        decode launches."""
        B = len(rs)
        c = self.cache
        t0 = time.perf_counter()
        end = np.ascontiguousarray(end, dtype=np.int32)
        cur32 = np.ascontiguousarray(cur, dtype=np.int32)
        run = np.zeros(max(B, 1), dtype=np.int32)
        nr = len(running)
        run[:nr] = running
        nodes = np.array([r.node for r in rs], dtype=np.int64)
        key = ("dec",) + tuple((r.rid, int(n)) for r, n in zip(rs, end))
        hit = self._match_cache.get(key)         # the same every pass: cached (a fresh multi-MB array
        if hit is None:                          # per batch costs page faults)
            tok_off = np.zeros(B + 1, dtype=np.int64)
            tok_off[1:] = np.cumsum(end)
            hit = self._match_cache[key] = (np.concatenate([r.tokens[:n] for r, n in zip(rs, end)]), tok_off)
        tokens, tok_off = hit
        collect = self.plan_only and self.collect_calls
        hcat = np.concatenate([r.hashes[:n] for r, n in zip(rs, end)]) if collect else None
        chunk = self.launch_chunk
        meta = np.zeros((chunk, 3), dtype=np.int64)
        events = self._step_events(rs) if self.record else None
        self.stats["tree_s"] += time.perf_counter() - t0
        while nr > 0:
            t0 = time.perf_counter()
            cap = 4 * nr * chunk
            if self.plan_only:
                stage, name = None, None
                sn = np.empty(cap, dtype=np.int32)
            else:
                name = f"dec{self._ring % 4}"
                self._ring += 1
                stage = self._pinned(name, cap)
                sn = stage.numpy()
            st, ns, nr = c.rx_decode_steps(slots, cur32, end, self._stable, nodes, tokens, tok_off, run, nr, chunk,
                                           sn, meta, events)
            m = meta[:ns].copy()
            self.stats["decode_tokens"] += int(m[:, 0].sum())
            if collect:
                for Bk, o, _ in m:
                    rows, seq = sn[o + 2 * Bk:o + 3 * Bk], sn[o + Bk:o + 2 * Bk]
                    self.calls.append(CallPlan("decode", hcat[tok_off[rows] + seq - 1], {"B": int(Bk)}))
            self.stats["tree_s"] += time.perf_counter() - t0
            if stage is not None:
                if ns:
                    self._decode_launch(stage[:int(m[-1, 1] + 4 * m[-1, 0])], name, m)
                else:
                    self._pinned_done(name)
            if st != 0:
                raise OutOfSlots(f"decode step needs {nr} slots, available {c.rx_available()}")

    def _step_events(self, rs):
        """rx_decode_steps event callback -> the same trace tuples as the Python path."""
        runs = []

        def ev(kind, v, s):
            if kind == 1:
                runs.append(tuple(int(x) for x in s))
            elif kind == 2:
                self._rec("evict", int(v[0]), int(v[1]), tuple(runs))
                runs.clear()
            elif kind == 0:
                self._rec("alloc", int(v[0]), tuple(int(x) for x in s))
            else:
                b = int(v[0])
                self._rec("dec_ref", rs[b].rid, int(v[1]))
                self._rec("insert", rs[b].rid, int(v[2]), int(v[3]))
        return ev

    def _output_loop_py(self, rs, slots, cur, running, nseg, unit):
        """Output phase in Python: jump-forward segments (FSM workload), DP workers (evictions go to
        the router as token paths) and the on_decode_plan hook.  Host ahead of the device: the tree
        ops of each step run on the host (none depends on GPU results), and every launch_chunk
        steps the planned steps are launched (runs of single-token steps as decode calls with ONE
        metadata H2D, multi-token steps as extend calls)."""
        step = 0
        steps = []
        while len(running):
            t0 = time.perf_counter()
            if unit:
                lens = np.ones(len(running), dtype=np.int64)
            else:
                lens = np.array([rs[b].segs[step] for b in running], dtype=np.int64)
            new = self._alloc(int(lens.sum()))
            pos = cur[running].copy()
            if (lens == 1).all():
                slots[running, pos] = new
                steps.append(("dec", running, new, pos))
                if self.on_decode_plan is not None:
                    self.on_decode_plan(self, slots, running, pos)
                if self.plan_only and self.collect_calls:
                    hs = np.array([rs[b].hashes[p_] for b, p_ in zip(running, pos)], dtype=np.uint64)
                    self.calls.append(CallPlan("decode", hs, {"B": len(running)}))
            else:
                slots.reshape(-1)[_ragged_flat(running.astype(np.int64) * slots.shape[1] + pos, lens)] = new
                steps.append(("ext", running, pos, lens))
                if self.plan_only and self.collect_calls:
                    hs = np.concatenate([rs[b].hashes[p_:p_ + n_] for b, p_, n_ in zip(running, pos, lens)])
                    self.calls.append(CallPlan("extend", hs.astype(np.uint64), {"ext": lens.tolist()}))
            cur[running] += lens
            self.stats["decode_tokens"] += int(lens.sum())
            step += 1
            done = nseg[running] <= step
            if done.any():
                self._finish_many(rs, running[done], slots)
            running = running[~done]
            self.stats["tree_s"] += time.perf_counter() - t0
            if len(steps) >= self.launch_chunk and not self.plan_only:
                self._launch_steps(rs, slots, steps)          # keep the GPU fed while the host plans on
                steps = []
        if steps and not self.plan_only:
            self._launch_steps(rs, slots, steps)

    def _launch_steps(self, rs, slots, steps):
        """Launch planned output steps in order: runs of decode steps share one metadata H2D."""
        i = 0
        while i < len(steps):
            if steps[i][0] == "ext":
                _, running, pos, lens = steps[i]
                self._extend_step(rs, slots, running, pos, lens)
                i += 1
                continue
            j = i
            while j < len(steps) and steps[j][0] == "dec":
                j += 1
            self._decode_phase([st[1:] for st in steps[i:j]])
            i = j

    def _finish_many(self, rs, idx, slots):
        """Alg. 1 finished requests: dec_ref then insert(prompt + outputs), in batch order,
        one C call for all of them."""
        if len(idx) == 0:
            return
        lens = np.array([rs[b].n_prompt + rs[b].n_out for b in idx], dtype=np.int64)
        off = np.zeros(len(idx) + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens)
        toks = np.concatenate([rs[b].tokens[:n] for b, n in zip(idx, lens)])
        if (lens == lens[0]).all():
            sl = slots[idx, :int(lens[0])].reshape(-1)
        else:
            sl = np.concatenate([slots[b, :n] for b, n in zip(idx, lens)])
        d, nc, nd = self.cache.rx_finish_batch([rs[b].node for b in idx], toks, off, sl)
        if self.record:
            for i, b in enumerate(idx):
                self._rec("dec_ref", rs[b].rid, int(d[i]))
                self._rec("insert", rs[b].rid, int(nc[i]), int(nd[i]))

    # ------------------------------------------------------------------ attention calls
    def _extend(self, rs, slots, prefix, ext):
        total = int(ext.sum())
        B = len(rs)
        self.stats["extend_tokens"] += total
        if self.plan_only:
            if not self.collect_calls:
                return
            hs = np.array([h for r, n in zip(rs, ext) for h in r.hashes[r.prefix:r.prefix + n]], dtype=np.uint64)
            self.calls.append(CallPlan("extend", hs, {"ext": ext.tolist(), "prefix": prefix.tolist()}))
            return
        self._extend_launch(slots, None, prefix, ext)

    def _extend_step(self, rs, slots, running, pos, lens):
        """A multi-token output step (jump forward): the running requests' segments
        (sampled token + forced edge) are processed by one extend call over their cached context
        (prefix = current length), table rows selected by `running`."""
        self._extend_launch(slots, running, pos, lens, shared=self._shared)

    def _extend_launch(self, slots, rows, prefix, ext, shared=0):
        """rx_extend over table `slots` (every row of the batch, uploaded whole so later decode
        steps index it by batch row); batch entry b uses row rows[b] (None = identity)."""
        dev = self.device
        B = len(prefix)
        total = int(ext.sum())
        q, k_new, v_new = self.bank.ext[self._ext_i]
        self._ext_i += 1
        R, stride = slots.shape
        name = f"ext{self._ext_ring % 8}"            # ring: the host may run several extends ahead
        self._ext_ring += 1
        # an output step (rows given) keeps the batch's device table and writes only its new slots
        # into it (rx_store_kv's table append); a prefill uploads the table whole
        incremental = rows is not None and self._rtt is not None and tuple(self._rtt.shape) == (R, stride)
        tail = 3 * total if incremental else R * stride
        hdr = 4 * (B + 1)
        stage = self._pinned(name, hdr + tail)
        sn = stage.numpy()
        sn[0:B] = prefix
        sn[B + 1:2 * B + 1] = ext
        sn[2 * B + 2] = 0
        sn[2 * B + 3:3 * B + 3] = np.cumsum(ext)
        if rows is not None:
            sn[3 * B + 3:4 * B + 3] = rows
        if incremental:
            # [int64 flat table index (2 int32 words each) | int32 slot] of every new row
            flat = _ragged_flat(np.asarray(rows, dtype=np.int64) * stride + prefix, ext)
            new_slots = slots.reshape(-1)[flat]
            o2 = hdr + (hdr & 1)                     # 8-byte alignment of the int64 block
            sn[o2:o2 + 2 * total].view(np.int64)[:] = flat
            sn[o2 + 2 * total:o2 + 3 * total] = new_slots
        else:
            sn[hdr:] = slots.reshape(-1)
        dstage = self._upload(stage)
        self._pinned_done(name)
        if incremental:
            d_idx = dstage[o2:o2 + 2 * total].view(torch.int64)
            d_new = dstage[o2 + 2 * total:o2 + 3 * total]
        else:
            self._rtt = dstage[hdr:].view(R, stride)
        ws_n = api.rx_decode_workspace_bytes(self.cfg, R, stride)
        if self._ws is None or self._ws.numel() < ws_n:
            self._ws = torch.zeros(max(ws_n, 256), dtype=torch.uint8, device=dev)   # >= the counter header (rx.h)
        o = torch.empty((total, self.hq, self.shape.head_dim), dtype=torch.bfloat16, device=dev)
        chunks = self._gather_chunks(ext) if (self.gather is not None and hasattr(self.gather, "start")) else None
        ev0 = self._tbeg()
        nl0 = 0
        if incremental:
            # table entries only: the rx_extend(_cascade) below stores the rows' K/V itself
            api.rx_store_kv(self.cfg, d_new, None, None, None, None, self._rtt, d_idx)
            nl0 = api.rx_last_launch_count()
        if chunks is None and shared > 0:
            # every row shares cached positions [0, shared): attend them once for all rows (cascade)
            ws_n = api.rx_extend_cascade_workspace_bytes(self.cfg, total, shared)
            if self._ws.numel() < ws_n:
                self._ws = torch.zeros(2 * ws_n, dtype=torch.uint8, device=dev)
            api.rx_extend_cascade(self.cfg, self._rtt, dstage[3 * B + 3:4 * B + 3] if rows is not None else None,
                                  dstage[0:B], dstage[B + 1:2 * B + 1], dstage[2 * B + 2:3 * B + 3], total,
                                  int(ext.max()), int(prefix.max()), shared, q, k_new, v_new, self.k_pool,
                                  self.v_pool, o, self._ws)
            nl = api.rx_last_launch_count()
        elif chunks is None:
            api.rx_extend(self.cfg, self._rtt, dstage[3 * B + 3:4 * B + 3] if rows is not None else None,
                          dstage[0:B], dstage[B + 1:2 * B + 1], dstage[2 * B + 2:3 * B + 3],
                          total, int(ext.max()), int(prefix.max()), q, k_new, v_new, self.k_pool, self.v_pool, o, self._ws)
            nl = api.rx_last_launch_count()
        else:
            # TP: the call runs as request blocks; each block's rows are all-gathered (async, NCCL
            # stream) while the next block computes (SURVEY §8(e) chunked overlap)
            nl = 0
            out = self.gather.alloc(total, self.hq, self.shape.head_dim, o.dtype, dev)
            handles = []
            cname = f"extc{self._ext_ring % 8}"
            cst = self._pinned(cname, 4 * (B + len(chunks)))
            cn = cst.numpy()
            o_ = 0
            meta = []
            for b0, b1 in chunks:
                n = b1 - b0
                cn[o_:o_ + n] = prefix[b0:b1]
                cn[o_ + n:o_ + 2 * n] = ext[b0:b1]
                cn[o_ + 2 * n] = 0
                cn[o_ + 2 * n + 1:o_ + 3 * n + 1] = np.cumsum(ext[b0:b1])
                cn[o_ + 3 * n + 1:o_ + 4 * n + 1] = rows[b0:b1] if rows is not None else np.arange(b0, b1)
                meta.append((o_, n))
                o_ += 4 * n + 1
            dchunk = self._upload(cst)
            self._pinned_done(cname)
            qo = np.concatenate([[0], np.cumsum(ext)])
            for (b0, b1), (c0, n) in zip(chunks, meta):
                r0, r1 = int(qo[b0]), int(qo[b1])
                if r1 == r0:
                    continue
                d = dchunk[c0:c0 + 4 * n + 1]
                api.rx_extend(self.cfg, self._rtt, d[3 * n + 1:4 * n + 1], d[0:n], d[n:2 * n], d[2 * n:3 * n + 1],
                              r1 - r0, int(ext[b0:b1].max()), int(prefix[b0:b1].max()), q[r0:r1], k_new[r0:r1],
                              v_new[r0:r1], self.k_pool, self.v_pool, o[r0:r1], self._ws)
                nl += api.rx_last_launch_count()
                handles.append(self.gather.start(o[r0:r1], out, r0, r1))
        self.stats["launches"] += nl + nl0
        if ev0 is not None:
            # algorithmic FLOPs: 4*hd*H_q*sum(n*p + n(n+1)/2), causal-masked work not counted
            n, p_ = ext.astype(np.float64), prefix.astype(np.float64)
            flops = 4.0 * self.shape.head_dim * self.hq * float(np.sum(n * p_ + n * (n + 1) / 2))
            self._tend(ev0, "extend", flops, nl)
        if chunks is not None:
            evg = self._tbeg()
            o = self.gather.finish(handles, out)
            if evg is not None:
                self._tend(evg, "gather", 0.0, 0)
        elif self.gather is not None:
            evg = self._tbeg()
            o = self.gather(o)
            if evg is not None:
                self._tend(evg, "gather", 0.0, 0)
        if self.sink is not None:
            self.sink("extend", o)
        if self.keep_outputs:
            self.outputs.append(("extend", o, {"ext": ext.tolist()}))

    def _gather_chunks(self, ext):
        """Request blocks of a TP extend call whose outputs are gathered while later blocks run:
        about gather_chunk_rows rows each; None when the call is small (one gather)."""
        total = int(ext.sum())
        if total < 2 * self.gather_chunk_rows:
            return None
        cum = np.cumsum(ext)
        cuts = np.searchsorted(cum, np.arange(self.gather_chunk_rows, total, self.gather_chunk_rows), side="left") + 1
        edges = [0] + sorted(set(int(c) for c in cuts if 0 < c < len(ext))) + [len(ext)]
        return [(edges[i], edges[i + 1]) for i in range(len(edges) - 1)] if len(edges) > 2 else None

    def _decode_phase(self, steps):
        """Launch a batch's decode steps planned in Python: their records [new slots | seq_lens | rows
        | stable lens] in one pinned staging buffer (the rx_decode_steps layout), then _decode_launch."""
        offs = np.zeros(len(steps) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([4 * len(r) for r, _, _ in steps])
        name = f"dec{self._ring % 4}"
        self._ring += 1
        stage = self._pinned(name, int(offs[-1]))
        sn = stage.numpy()
        meta = np.zeros((len(steps), 3), dtype=np.int64)
        for k, ((running, new, pos), o0) in enumerate(zip(steps, offs)):
            B = len(running)
            sn[o0:o0 + B] = new
            sn[o0 + B:o0 + 2 * B] = pos + 1             # seq_len counts the new token
            sn[o0 + 2 * B:o0 + 3 * B] = running         # table row of each running request
            sn[o0 + 3 * B:o0 + 4 * B] = self._stable[running]   # written by the batch's prefill
            meta[k] = (B, o0, int(pos.max()) + 1)
        self._decode_launch(stage, name, meta)

    def _decode_launch(self, stage, name, meta):
        """One H2D of the staged step records, then one rx_decode_append (or
        rx_decode_cascade_append) per step.  meta[k] = (B, word offset, max seq_len)."""
        dev = self.device
        sh = self._shared
        need = 0
        for B, _, ms in meta:
            need = max(need, api.rx_decode_cascade_workspace_bytes(self.cfg, int(B), int(ms), sh) if sh
                       else api.rx_decode_workspace_bytes(self.cfg, int(B), int(ms)))
        # decode_bytes() needs (running, pos) per call, read after the timed region: copy the records
        sn = stage.numpy().copy() if self.timer is not None else None
        d_all = self._upload(stage)
        self._pinned_done(name)
        if need > self._ws.numel():
            self._ws = torch.zeros(2 * need, dtype=torch.uint8, device=dev)   # geometric growth
        # timing: one event pair around the whole run of back-to-back decode calls (per-call events
        # on ~2000 calls per C3 step would perturb the step); per call when outputs are gathered
        # (TP), so the all-gather stays outside the kernel brackets
        # TP with the gather fused into the epilogue (tp.FusedGather): the calls store straight into
        # every rank's gathered buffer; one flag barrier ends the run, then the outputs are read
        fused = getattr(self.gather, "fused", False)
        per_call = self.gather is not None and not fused
        if (self.gather is None or fused) and not _PER_STEP_LAUNCH:
            self._decode_run_native(d_all, sn, meta, sh, fused)
            return
        ev_run = None if per_call else self._tbeg()
        works, nl_run, pending = [], 0, []
        if fused:
            self.gather.begin_run()
        for B, o0, max_seq in meta:
            B, o0, max_seq = int(B), int(o0), int(max_seq)
            q, k, v = self.bank.dec[self._dec_i]
            self._dec_i += 1
            d = d_all[o0:o0 + 4 * B]
            ev0 = self._tbeg() if per_call else None
            if fused:
                hq_all, hd = self.shape.h_q, self.shape.head_dim
                if not self.gather.fits(B, hq_all, hd):   # region full: end the run, start the next
                    self._fused_end_run(pending)
                    pending = []
                    self.gather.begin_run()
                dests, o = self.gather.take(B, hq_all, hd)
                out = api.tp_out(dests, hq_all, int(self.heads_q[0]))
                api.rx_decode_append_tp(self.cfg, self._rtt, d[2 * B:3 * B], d[B:2 * B], max_seq, sh, q, k, v,
                                        d[:B], self.k_pool, self.v_pool, out, self._ws, stable_lens=d[3 * B:])
            else:
                o = torch.empty((B, self.hq, self.shape.head_dim), dtype=torch.bfloat16, device=dev)
            if fused:
                pass
            elif sh:
                # the suffix decode reads its stable positions (the prompt) while the previous step's
                # merge drains, and releases the shared pass only after its streaming (that kernel
                # needs whole SMs: releasing it early measured slower, C5 step 101 -> 140 us)
                api.rx_decode_cascade_append(self.cfg, self._rtt, d[2 * B:3 * B], d[B:2 * B], max_seq, sh, q, k, v,
                                             d[:B], self.k_pool, self.v_pool, o, self._ws,
                                             stable_lens=None if _NO_CAS_STABLE else d[3 * B:])
            else:
                api.rx_decode_append(self.cfg, self._rtt, d[2 * B:3 * B], d[B:2 * B], max_seq, q, k, v, d[:B],
                                     self.k_pool, self.v_pool, o, self._ws, stable_lens=d[3 * B:])
            nl = api.rx_last_launch_count()
            self.stats["launches"] += nl
            if sn is not None:
                # algorithmic bytes: distinct pool rows read (K+V) + q + o + slot
                # indices, computed after the timed region from (slots, running, pos)
                w = (self._slots_host, sn[o0 + 2 * B:o0 + 3 * B].astype(np.int64), sn[o0 + B:o0 + 2 * B] - 1)
                if ev0 is not None:
                    self._tend(ev0, "decode", [w], nl)
                works.append(w)
            nl_run += nl
            if fused:
                pending.append((o, B))
                continue
            if self.gather is not None:
                evg = self._tbeg()
                o = self.gather(o)
                if evg is not None:
                    self._tend(evg, "gather", 0.0, 0)
            if self.sink is not None:
                self.sink("decode", o)
            if self.keep_outputs:
                self.outputs.append(("decode", o, {"B": B}))
        if ev_run is not None:
            self._tend(ev_run, "decode", works, nl_run, calls=len(meta))
        if fused:
            self._fused_end_run(pending)

    def _decode_run_native(self, d_all, sn, meta, sh, fused=False):
        """The run's steps in as few library calls as possible (rx_decode_run): per-step host cost
        is the C launch path only (a Python call per step cost ~35-48 us of host time, more than a
        cascade step's device time on C2 / C4).  Outputs are consecutive views of one buffer, or
        (fused TP gather) of the gather's region on every rank."""
        dev, hd = self.device, self.shape.head_dim
        ev_run = self._tbeg()
        n = len(meta)
        Bs = [int(B) for B, _, _ in meta]
        o_all = None if fused else torch.empty((sum(Bs), self.hq, hd), dtype=torch.bfloat16, device=dev)
        hq_all = self.shape.h_q
        # host-resident inputs (hostio._BlockPrefetcher) hand out a block's ring slot for reuse when
        # the first call of the NEXT block is taken, i.e. they expect a block's kernels enqueued by
        # then: a library call never crosses a block boundary; device banks: one call per run
        blk = getattr(self.bank.dec, "block", None)
        outs, pending, nl, r = [], [], 0, 0
        chunk = {"k": [], "q": [], "k_": [], "v": [], "o": []}

        def flush():
            nonlocal nl
            ks_ = chunk["k"]
            if not ks_:
                return
            api.rx_decode_run(self.cfg, self._rtt, d_all, [int(meta[k][1]) for k in ks_], [Bs[k] for k in ks_],
                              [int(meta[k][2]) for k in ks_], sh, chunk["q"], chunk["k_"], chunk["v"], self.k_pool,
                              self.v_pool, chunk["o"], self._ws, with_stable=not (sh and _NO_CAS_STABLE),
                              tp=(hq_all, int(self.heads_q[0])) if fused else None)
            nl += api.rx_last_launch_count()
            for key in chunk:
                chunk[key] = []

        if fused:
            self.gather.begin_run()
        for k in range(n):
            B = Bs[k]
            if blk is not None and self._dec_i % blk == 0:
                flush()
            if fused and not self.gather.fits(B, hq_all, hd):   # region full: end the run, start the next
                flush()
                self._fused_end_run(pending)
                pending = []
                self.gather.begin_run()
            q, kk, v = self.bank.dec[self._dec_i]
            self._dec_i += 1
            if fused:
                dests, o = self.gather.take(B, hq_all, hd)
                chunk["o"].append(dests)
                pending.append((o, B))
            else:
                o = o_all[r:r + B]
                r += B
                chunk["o"].append(o)
                outs.append(o)
            chunk["k"].append(k)
            chunk["q"].append(q)
            chunk["k_"].append(kk)
            chunk["v"].append(v)
        flush()
        self.stats["launches"] += nl
        works = []
        if sn is not None:
            # algorithmic bytes: distinct pool rows read (K+V) + q + o + slot indices,
            # computed after the timed region from (slots, running, pos)
            for B, o0, _ in meta:
                B, o0 = int(B), int(o0)
                works.append((self._slots_host, sn[o0 + 2 * B:o0 + 3 * B].astype(np.int64), sn[o0 + B:o0 + 2 * B] - 1))
        if ev_run is not None:
            self._tend(ev_run, "decode", works, nl, calls=n)
        if fused:
            self._fused_end_run(pending)
            return
        for o, B in zip(outs, Bs):
            if self.sink is not None:
                self.sink("decode", o)
            if self.keep_outputs:
                self.outputs.append(("decode", o, {"B": B}))

    def _fused_end_run(self, pending):
        """End a FusedGather run: the host sink's copies of the previous run are done (a peer may
        overwrite that region after this barrier), the barrier (every rank's stores of this run are
        visible here), then this run's gathered outputs go to the sink / the kept outputs."""
        if self.sink is not None and hasattr(self.sink, "join"):
            self.sink.join()
        evg = self._tbeg()
        self.gather.end_run()
        if evg is not None:
            self._tend(evg, "gather", 0.0, 1)
        for o, B in pending:
            if self.sink is not None:
                self.sink("decode", o)
            if self.keep_outputs:
                self.outputs.append(("decode", o.clone(), {"B": B}))

    # ------------------------------------------------------------------ pinned staging
    def _upload(self, stage):
        """Device copy of a pinned staging slice, made by an SM kernel (rx_copy_h2d): metadata uploads
        must not wait on the copy engines behind a large input prefetch (e2e path)."""
        d = torch.empty(stage.shape, dtype=stage.dtype, device=self.device)
        api.rx_copy_h2d(d, stage)
        self.stats["launches"] += 1
        return d

    def _pinned(self, name, n):
        """Pinned int32 staging buffer of >= n elements from a pool: the oldest buffer that is large
        enough and whose last H2D copy has completed is reused, so steady state allocates nothing —
        pinned allocation (cudaHostAlloc) takes milliseconds.  `name` tags the checkout."""
        pool = self._pin_pool                 # oldest first: the first entries are the ones done
        pick = None
        for i, (buf, ev) in enumerate(pool):
            if buf.numel() >= n and ev.query():
                pick = i
                break
        if pick is None:
            buf = torch.empty(max(n, 1 << 16), dtype=torch.int32, pin_memory=True)
        else:
            buf, _ = pool.pop(pick)
        self._pin_cache[name] = buf
        return buf[:n]

    def _pinned_done(self, name):
        """The H2D copy from the buffer checked out as `name` is enqueued: return it to the pool,
        reusable once that copy has run."""
        buf = self._pin_cache.pop(name)
        ev = torch.cuda.Event()
        ev.record()
        self._pin_pool.append((buf, ev))

    # ------------------------------------------------------------------ timing hooks
    def enable_timing(self, on=True):
        self.timer = [] if on else None

    def _tbeg(self):
        if self.timer is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def _tend(self, ev0, kind, work, launches, calls=1):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.timer.append((kind, ev0, e, work, launches, calls))

    def decode_bytes(self, work):
        """(algorithmic, logical) bytes of one rx_decode call: distinct pool rows read once (K+V),
        plus q, o and the slot indices; logical counts every request's rows."""
        slots, running, pos = work
        hd, B = self.shape.head_dim, len(running)
        L = int(pos.max()) + 1
        mask = np.arange(L)[None, :] <= pos[:, None]
        uniq = np.unique(slots[running][:, :L][mask]).size
        extra = 2 * B * self.hq * hd * 2 + 4 * int((pos + 1).sum())
        row = self.hkv * hd * 2 * 2
        return float(uniq * row + extra), float(int((pos + 1).sum()) * row + extra)

    def timing_summary(self):
        """{kind: [total ms, launches, calls, total work, logical work]} from the recorded events (call
        after a sync).  work = FLOPs (extend) or algorithmic bytes (decode: distinct pool rows once);
        logical = the same for extend, every request's rows for decode (paged-equivalent bytes)."""
        out = {}
        for kind, a, b, work, nl, calls in self.timer or []:
            ms = a.elapsed_time(b)
            t = out.setdefault(kind, [0.0, 0, 0, 0.0, 0.0])
            t[0] += ms
            t[1] += nl
            t[2] += calls
            if kind == "decode":
                for w in work:
                    alg, logical = self.decode_bytes(w)
                    t[3] += alg
                    t[4] += logical
            else:
                t[3] += work
                t[4] += work
        return out

    # ------------------------------------------------------------------ workloads
    def reset(self):
        """Fresh tree + slot pool for another pass; device pools and the input bank are kept."""
        self.cache.close()
        self.cache = api.RadixCache(self.wl.num_slots)
        self.trace = []
        self.outputs = []
        self._ext_i = self._dec_i = 0
        self._slot_buf_i = 0
        for k in ("prompt_tokens", "cached_prompt_tokens", "extend_tokens", "decode_tokens", "output_tokens",
                  "launches"):
            self.stats[k] = 0
        self.stats["tree_s"] = 0.0

    def run_workload(self, bank: InputBank | None = None):
        if not self.plan_only:
            assert bank is not None, "execute pass needs an InputBank (build it from a plan pass)"
            self.bank = bank
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
            hist = [np.asarray(r.tokens, dtype=np.int32) for r in done]
        return self

    def _run_tot(self):
        """C4 tree-of-thought: root as a hint, then each level's branches under Alg. 1 admission."""
        from rxgen.workloads import Request
        m = self.wl.meta
        root = np.asarray(m["root"], dtype=np.int32)
        self.run_batch([Request(root, 0, "root")])
        parents = [root]
        for lvl, nodes in enumerate(m["levels"]):
            reqs = [Request(np.concatenate([parents[p], bp]), tl, f"L{lvl}n{i}") for i, (p, bp, tl) in enumerate(nodes)]
            parents = [np.asarray(r.tokens, dtype=np.int32) for r in self.run_waves(reqs)]
        return self


def plan_and_bank(wl, device="cuda", tp_rank=0, tp_size=1, q_scale=1.0, policy="lspf", host_gen=False):
    """Plan pass + input generation (untimed setup).  Returns (plan engine, InputBank)."""
    plan = Engine(wl, device=device, tp_rank=tp_rank, tp_size=tp_size, plan_only=True, policy=policy)
    plan.run_workload()
    bank = InputBank(plan.calls, wl.shape, plan.heads_q, plan.heads_kv, device, q_scale=q_scale, host=host_gen)
    return plan, bank
