"""Python binding of librx.so: same names as include/rx.h, argument marshalling only.

* ``RadixCache`` wraps ``rx_cache`` (host radix tree + token-slot pool).
* ``rx_store_kv`` / ``rx_extend`` / ``rx_decode`` take torch CUDA tensors and
  launch on the current torch stream.  Every step runs in librx's kernels;
  torch supplies device memory and the stream only.  Wrong device / dtype /
  layout raises — there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._lib import lib, AttnCfg, TpOut, EVICT_CB, EVICT_PATH_CB, STEP_EVENT_CB, RxError, P32, P64

_I32 = np.int32
SCHED_POLICY = {"lspf": 0, "fcfs": 1, "random": 2}   # rx_sched_policy


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=_I32)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(P32)


def _check(st: int, what: str):
    if st != 0:
        raise RxError(st, what)


class RadixCache:
    """rx_cache: the radix tree and the token-slot pool it shares with running requests."""

    def __init__(self, num_slots: int):
        h = C.c_void_p()
        _check(lib.rx_cache_create(num_slots, C.byref(h)), "rx_cache_create")
        self._h = h
        self.num_slots = num_slots
        self._runs = []
        self._cb = EVICT_CB(self._on_evict)

    def close(self):
        if self._h:
            lib.rx_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _on_evict(self, user, slots, n):
        self._runs.append(np.ctypeslib.as_array(slots, shape=(n,)).copy() if n else np.zeros(0, _I32))

    # -------------------------------------------------------------- tree
    def rx_match_prefix(self, tokens):
        """-> (node handle, matched_len, slots int32[matched_len])"""
        t = _i32(tokens)
        out = np.empty(max(len(t), 1), dtype=_I32)
        node, m = C.c_int64(), C.c_int64()
        _check(lib.rx_match_prefix(self._h, _p32(t), len(t), C.byref(node), C.byref(m), _p32(out)),
               "rx_match_prefix")
        return node.value, m.value, out[:m.value]

    def rx_insert(self, tokens, slots):
        """-> (new_cached, dup_freed)"""
        t, s = _i32(tokens), _i32(slots)
        if len(t) != len(s):
            raise ValueError("tokens/slots length mismatch")
        nc, nd = C.c_int64(), C.c_int64()
        _check(lib.rx_insert(self._h, _p32(t), _p32(s), len(t), C.byref(nc), C.byref(nd)), "rx_insert")
        return nc.value, nd.value

    def rx_inc_ref(self, node: int) -> int:
        d = C.c_int64()
        _check(lib.rx_inc_ref(self._h, node, C.byref(d)), "rx_inc_ref")
        return d.value

    def rx_dec_ref(self, node: int) -> int:
        d = C.c_int64()
        _check(lib.rx_dec_ref(self._h, node, C.byref(d)), "rx_dec_ref")
        return d.value

    def rx_evict(self, needed: int):
        """-> (evicted tokens, [slot runs in eviction order])"""
        self._runs = []
        ev = C.c_int64()
        _check(lib.rx_evict(self._h, needed, C.byref(ev), self._cb, None), "rx_evict")
        return ev.value, self._runs

    def rx_evict_paths(self, needed: int):
        """-> (evicted, [(path tokens, leaf_start, slots)] in eviction order)"""
        out = []

        def cb(user, path, plen, leaf_start, slots, n):
            out.append((np.ctypeslib.as_array(path, shape=(plen,)).copy(), int(leaf_start),
                        np.ctypeslib.as_array(slots, shape=(n,)).copy() if n else np.zeros(0, _I32)))

        f = EVICT_PATH_CB(cb)
        ev = C.c_int64()
        _check(lib.rx_evict_paths(self._h, needed, C.byref(ev), f, None), "rx_evict_paths")
        return ev.value, out

    def rx_alloc(self, n: int):
        """n smallest free slots (ascending) or None on RX_E_NOMEM."""
        out = np.empty(max(n, 1), dtype=_I32)
        st = lib.rx_alloc(self._h, n, _p32(out))
        if st == -2:
            return None
        _check(st, "rx_alloc")
        return out[:n]

    def rx_alloc_evict(self, n: int):
        """Alg. 1 alloc -> evict shortfall -> retry.  -> (slots or None, evicted, runs)"""
        self._runs = []
        out = np.empty(max(n, 1), dtype=_I32)
        ev = C.c_int64()
        st = lib.rx_alloc_evict(self._h, n, _p32(out), C.byref(ev), self._cb, None)
        if st == -2:
            return None, ev.value, self._runs
        _check(st, "rx_alloc_evict")
        return out[:n], ev.value, self._runs

    def rx_free(self, slots):
        s = _i32(slots)
        _check(lib.rx_free(self._h, _p32(s), len(s)), "rx_free")

    # -------------------------------------------------------------- batched (one C call per step)
    def rx_match_prefix_batch(self, tokens_concat, offsets, out=None):
        """-> (nodes int64[B], matched int64[B], slots int32 (same layout as tokens_concat)); `out`: an
        int32 buffer of >= len(tokens_concat) entries to write the slots into (reused by the caller:
        a fresh multi-MB array per call costs page faults)"""
        t = _i32(tokens_concat)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        B = len(off) - 1
        nodes = np.empty(B, dtype=np.int64)
        matched = np.empty(B, dtype=np.int64)
        if out is not None and out.dtype == _I32 and out.flags.c_contiguous and len(out) >= max(len(t), 1):
            slots = out[:max(len(t), 1)]
        else:
            slots = np.empty(max(len(t), 1), dtype=_I32)
        _check(lib.rx_match_prefix_batch(self._h, B, _p32(t), off.ctypes.data_as(P64), nodes.ctypes.data_as(P64),
                                         matched.ctypes.data_as(P64), _p32(slots)), "rx_match_prefix_batch")
        return nodes, matched, slots

    def rx_inc_ref_batch(self, nodes):
        n = np.ascontiguousarray(nodes, dtype=np.int64)
        d = np.empty(len(n), dtype=np.int64)
        _check(lib.rx_inc_ref_batch(self._h, len(n), n.ctypes.data_as(P64), d.ctypes.data_as(P64)),
               "rx_inc_ref_batch")
        return d

    def rx_decode_steps(self, table, cur, end, stable, nodes, tokens, offsets, running, n_running, max_steps,
                        out, step_meta, events=None):
        """Alg. 1 output loop for plain decoding (rx.h rx_decode_steps).  table / cur / running / out /
        step_meta are updated IN PLACE (int32 C-contiguous; step_meta int64 [max_steps, 3]).
        events: callable(kind, vals int64 array, slots int32 array) or None.
        -> (status, n_steps, n_running); status 0 or RX_E_NOMEM (-2), other errors raise."""
        for a, dt in ((table, _I32), (cur, _I32), (running, _I32), (out, _I32), (step_meta, np.int64)):
            if a.dtype != dt or not a.flags.c_contiguous:
                raise ValueError("rx_decode_steps: in-place arrays must be C-contiguous of the declared dtype")
        if table.ndim != 2 or step_meta.size < 3 * max_steps:
            raise ValueError("rx_decode_steps: table must be [batch, stride], step_meta >= 3 * max_steps")
        e, st_, t = _i32(end), _i32(stable), _i32(tokens)
        nd = np.ascontiguousarray(nodes, dtype=np.int64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        nr, ns = C.c_int32(n_running), C.c_int32(0)
        cb = None
        if events is not None:
            def relay(user, kind, vals, slots, n):
                nv = {0: 1, 1: 0, 2: 2, 3: 4}[kind]
                v = np.ctypeslib.as_array(vals, shape=(nv,)).copy() if nv else np.zeros(0, np.int64)
                s = np.ctypeslib.as_array(slots, shape=(n,)).copy() if n else np.zeros(0, _I32)
                events(kind, v, s)
            cb = STEP_EVENT_CB(relay)
        st = lib.rx_decode_steps(self._h, len(cur), _p32(table), table.shape[1], _p32(cur), _p32(e), _p32(st_),
                                 nd.ctypes.data_as(P64), _p32(t), off.ctypes.data_as(P64), _p32(running),
                                 C.byref(nr), max_steps, _p32(out), out.size, step_meta.ctypes.data_as(P64),
                                 C.byref(ns), cb if cb is not None else STEP_EVENT_CB(), None)
        if st not in (0, -2):
            _check(st, "rx_decode_steps")
        return st, ns.value, nr.value

    def rx_finish_batch(self, nodes, tokens_concat, offsets, slots_concat):
        """dec_ref + insert per request -> (d_evict, new_cached, dup_freed), each int64[B]"""
        n = np.ascontiguousarray(nodes, dtype=np.int64)
        t, s = _i32(tokens_concat), _i32(slots_concat)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        B = len(n)
        d, nc, nd = (np.empty(B, dtype=np.int64) for _ in range(3))
        _check(lib.rx_finish_batch(self._h, B, n.ctypes.data_as(P64), _p32(t), off.ctypes.data_as(P64), _p32(s),
                                   d.ctypes.data_as(P64), nc.ctypes.data_as(P64), nd.ctypes.data_as(P64)),
               "rx_finish_batch")
        return d, nc, nd

    def rx_schedule(self, tokens_concat, offsets, max_new, policy="lspf", keys=None):
        """Alg. 1 admission step -> (nodes int64[B], matched int64[B], slots int32 (tokens layout),
        admitted int32[k] in admission order, deltas int64[k])."""
        t = _i32(tokens_concat)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        B = len(off) - 1
        mn = np.ascontiguousarray(max_new, dtype=np.int64)
        pol = SCHED_POLICY[policy]
        kp = None
        if keys is not None:
            keys = np.ascontiguousarray(keys, dtype=np.uint64)
            kp = keys.ctypes.data_as(C.POINTER(C.c_uint64))
        nodes, matched = np.empty(B, dtype=np.int64), np.empty(B, dtype=np.int64)
        slots = np.empty(max(len(t), 1), dtype=_I32)
        adm, d = np.empty(max(B, 1), dtype=_I32), np.empty(max(B, 1), dtype=np.int64)
        k = C.c_int32(0)
        _check(lib.rx_schedule(self._h, B, _p32(t), off.ctypes.data_as(P64), mn.ctypes.data_as(P64), pol, kp,
                               nodes.ctypes.data_as(P64), matched.ctypes.data_as(P64), _p32(slots), _p32(adm),
                               C.byref(k), d.ctypes.data_as(P64)), "rx_schedule")
        return nodes, matched, slots, adm[:k.value].copy(), d[:k.value].copy()

    def rx_evictable_size(self) -> int:
        return lib.rx_evictable_size(self._h)

    def rx_total_cached(self) -> int:
        return lib.rx_total_cached(self._h)

    def rx_available(self) -> int:
        return lib.rx_available(self._h)

    def rx_clock(self) -> int:
        return lib.rx_clock(self._h)

    def rx_dump_json(self) -> dict:
        n = lib.rx_dump_json(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib.rx_dump_json(self._h, buf, n + 1)
        return json.loads(buf.value.decode())


class Fsm:
    """rx_fsm: minimal DFA of a regex with compressed (singular) edges (§4, App. B)."""

    def __init__(self, regex: str):
        b = regex.encode("ascii")
        h = C.c_void_p()
        _check(lib.rx_fsm_create(b, len(b), C.byref(h)), "rx_fsm_create")
        self._h = h
        self.num_states = lib.rx_fsm_num_states(h)
        self._buf = (C.c_uint8 * 128)()

    def close(self):
        if self._h:
            lib.rx_fsm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rx_fsm_step(self, state: int, byte: int) -> int:
        return lib.rx_fsm_step(self._h, state, byte)

    def rx_fsm_is_accepting(self, state: int) -> bool:
        return lib.rx_fsm_is_accepting(self._h, state) == 1

    def rx_fsm_allowed(self, state: int):
        k = lib.rx_fsm_allowed(self._h, state, self._buf)
        return list(self._buf[:k])

    def rx_fsm_jump(self, state: int):
        """-> (forced bytes, end state)"""
        n = lib.rx_fsm_jump(self._h, state, None, 1 << 30, None)
        buf = (C.c_uint8 * max(n, 1))()
        end = C.c_int32()
        n = lib.rx_fsm_jump(self._h, state, buf, n, C.byref(end))
        return list(buf[:n]), end.value


class Router:
    """rx_router: the data-parallel meta-tree router (App. A.4)."""

    def __init__(self, num_workers: int):
        h = C.c_void_p()
        _check(lib.rx_router_create(num_workers, C.byref(h)), "rx_router_create")
        self._h = h
        self.num_workers = num_workers

    def close(self):
        if self._h:
            lib.rx_router_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def rx_router_affinity(self, tokens):
        t = _i32(tokens)
        aff = np.empty(self.num_workers, dtype=np.int64)
        _check(lib.rx_router_affinity(self._h, _p32(t), len(t), aff.ctypes.data_as(P64)), "rx_router_affinity")
        return aff

    def rx_router_dispatch(self, requests, loads, load_weight: float):
        """requests: list of token arrays; loads: int64 [W] (updated in place) -> (workers, affinities)"""
        t = _i32(np.concatenate([np.asarray(r, dtype=np.int32) for r in requests]) if len(requests)
                 else np.zeros(0, np.int32))
        off = np.zeros(len(requests) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(r) for r in requests])
        if not isinstance(loads, np.ndarray) or loads.dtype != np.int64 or not loads.flags.c_contiguous:
            raise ValueError("loads must be a contiguous int64 numpy array (updated in place)")
        w = np.empty(len(requests), dtype=_I32)
        a = np.empty(len(requests), dtype=np.int64)
        _check(lib.rx_router_dispatch(self._h, len(requests), _p32(t), off.ctypes.data_as(P64),
                                      loads.ctypes.data_as(P64), float(load_weight), _p32(w), a.ctypes.data_as(P64)),
               "rx_router_dispatch")
        return w, a

    def rx_router_insert(self, worker: int, tokens):
        t = _i32(tokens)
        _check(lib.rx_router_insert(self._h, worker, _p32(t), len(t)), "rx_router_insert")

    def rx_router_queue_evict(self, worker: int, path, leaf_start: int):
        t = _i32(path)
        _check(lib.rx_router_queue_evict(self._h, worker, _p32(t), len(t), leaf_start), "rx_router_queue_evict")

    def rx_router_sync(self) -> int:
        return lib.rx_router_sync(self._h)

    def rx_router_queue_len(self) -> int:
        return lib.rx_router_queue_len(self._h)

    def rx_router_dump_json(self) -> dict:
        n = lib.rx_router_dump_json(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        lib.rx_router_dump_json(self._h, buf, n + 1)
        return json.loads(buf.value.decode())


# ------------------------------------------------------------------ device calls
def attn_cfg(h_q: int, h_kv: int, head_dim: int, sm_scale: float) -> AttnCfg:
    return AttnCfg(h_q, h_kv, head_dim, sm_scale)


def _dev(t, dtype=None, name="tensor"):
    import torch
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def rx_store_kv(cfg: AttnCfg, slots, k, v, k_pool, v_pool, rtt=None, rtt_index=None, stream=None):
    import torch
    n = slots.shape[0]
    st = lib.rx_store_kv(C.byref(cfg), n, _dev(slots, torch.int32, "slots"), _dev(k, torch.bfloat16, "k"),
                         _dev(v, torch.bfloat16, "v"), _dev(k_pool, torch.bfloat16, "k_pool"),
                         _dev(v_pool, torch.bfloat16, "v_pool"), k_pool.shape[0] if k_pool is not None else 1,
                         _dev(rtt, torch.int32, "rtt"), _dev(rtt_index, torch.int64, "rtt_index"), _stream(stream))
    _check(st, "rx_store_kv")


def rx_extend_workspace_bytes(cfg: AttnCfg, batch: int, max_extend_len: int) -> int:
    return lib.rx_extend_workspace_bytes(C.byref(cfg), batch, max_extend_len)


def rx_decode_workspace_bytes(cfg: AttnCfg, batch: int, max_seq_len: int) -> int:
    return lib.rx_decode_workspace_bytes(C.byref(cfg), batch, max_seq_len)


def rx_extend(cfg: AttnCfg, rtt, rows, prefix_lens, extend_lens, qo_indptr, total_new: int, max_extend_len: int,
              max_prefix_len: int, q, k_new, v_new, k_pool, v_pool, o, ws=None, stream=None):
    """ws=None: a zeroed workspace of rx_extend_workspace_bytes is allocated (through torch) for this
    call; callers that issue many calls pass one zero-initialised buffer (include/rx.h "Workspaces")."""
    import torch
    batch = prefix_lens.shape[0]
    if ws is None:
        ws = torch.zeros(max(1, rx_extend_workspace_bytes(cfg, batch, max_extend_len)), dtype=torch.uint8,
                         device=q.device)
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_extend(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                       _dev(rows, torch.int32, "rows"), _dev(prefix_lens, torch.int32, "prefix_lens"),
                       _dev(extend_lens, torch.int32, "extend_lens"), _dev(qo_indptr, torch.int32, "qo_indptr"),
                       total_new, max_extend_len, max_prefix_len, _dev(q, torch.bfloat16, "q"),
                       _dev(k_new, torch.bfloat16, "k_new"), _dev(v_new, torch.bfloat16, "v_new"),
                       _dev(k_pool, torch.bfloat16, "k_pool"), _dev(v_pool, torch.bfloat16, "v_pool"),
                       k_pool.shape[0], _dev(o, torch.bfloat16, "o"), _dev(ws, None, "ws"), ws_bytes,
                       _stream(stream))
    _check(st, "rx_extend")


def rx_extend_cascade_workspace_bytes(cfg: AttnCfg, total_new: int, shared_len: int) -> int:
    return lib.rx_extend_cascade_workspace_bytes(C.byref(cfg), total_new, shared_len)


def rx_extend_cascade(cfg: AttnCfg, rtt, rows, prefix_lens, extend_lens, qo_indptr, total_new: int,
                      max_extend_len: int, max_prefix_len: int, shared_len: int, q, k_new, v_new, k_pool, v_pool, o,
                      ws=None, stream=None):
    """rx_extend with the rows' common cached prefix [0, shared_len) attended once (include/rx.h)."""
    import torch
    batch = prefix_lens.shape[0]
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_extend_cascade(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                               _dev(rows, torch.int32, "rows"), _dev(prefix_lens, torch.int32, "prefix_lens"),
                               _dev(extend_lens, torch.int32, "extend_lens"), _dev(qo_indptr, torch.int32, "qo_indptr"),
                               total_new, max_extend_len, max_prefix_len, shared_len, _dev(q, torch.bfloat16, "q"),
                               _dev(k_new, torch.bfloat16, "k_new"), _dev(v_new, torch.bfloat16, "v_new"),
                               _dev(k_pool, torch.bfloat16, "k_pool"), _dev(v_pool, torch.bfloat16, "v_pool"),
                               k_pool.shape[0], _dev(o, torch.bfloat16, "o"), _dev(ws, None, "ws"), ws_bytes,
                               _stream(stream))
    _check(st, "rx_extend_cascade")


def rx_decode(cfg: AttnCfg, rtt, rows, seq_lens, max_seq_len: int, q, k_pool, v_pool, o, ws=None, stream=None):
    import torch
    batch = seq_lens.shape[0]
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_decode(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                       _dev(rows, torch.int32, "rows"), _dev(seq_lens, torch.int32, "seq_lens"), max_seq_len,
                       _dev(q, torch.bfloat16, "q"), _dev(k_pool, torch.bfloat16, "k_pool"),
                       _dev(v_pool, torch.bfloat16, "v_pool"), k_pool.shape[0], _dev(o, torch.bfloat16, "o"),
                       _dev(ws, None, "ws"), ws_bytes, _stream(stream))
    _check(st, "rx_decode")


def rx_decode_append(cfg: AttnCfg, rtt, rows, seq_lens, max_seq_len: int, q, k_new, v_new, new_slots, k_pool,
                     v_pool, o, ws=None, stream=None, stable_lens=None):
    """rx_store_kv + rtt append + rx_decode of one decode step, in one kernel (include/rx.h)."""
    import torch
    batch = seq_lens.shape[0]
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_decode_append(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                              _dev(rows, torch.int32, "rows"), _dev(seq_lens, torch.int32, "seq_lens"),
                              _dev(stable_lens, torch.int32, "stable_lens"), max_seq_len,
                              _dev(q, torch.bfloat16, "q"), _dev(k_new, torch.bfloat16, "k_new"),
                              _dev(v_new, torch.bfloat16, "v_new"), _dev(new_slots, torch.int32, "new_slots"),
                              _dev(k_pool, torch.bfloat16, "k_pool"), _dev(v_pool, torch.bfloat16, "v_pool"),
                              k_pool.shape[0], _dev(o, torch.bfloat16, "o"), _dev(ws, None, "ws"), ws_bytes,
                              _stream(stream))
    _check(st, "rx_decode_append")


def rx_decode_cascade_workspace_bytes(cfg: AttnCfg, batch: int, max_seq_len: int, shared_len: int) -> int:
    return lib.rx_decode_cascade_workspace_bytes(C.byref(cfg), batch, max_seq_len, shared_len)


def rx_decode_cascade_append(cfg: AttnCfg, rtt, rows, seq_lens, max_seq_len: int, shared_len: int, q, k_new, v_new,
                             new_slots, k_pool, v_pool, o, ws=None, stream=None, stable_lens=None):
    """Shared-prefix decode step (include/rx.h rx_decode_cascade_append)."""
    import torch
    batch = seq_lens.shape[0]
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_decode_cascade_append(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                                      _dev(rows, torch.int32, "rows"), _dev(seq_lens, torch.int32, "seq_lens"),
                                      _dev(stable_lens, torch.int32, "stable_lens"), max_seq_len, shared_len,
                                      _dev(q, torch.bfloat16, "q"),
                                      _dev(k_new, torch.bfloat16, "k_new"), _dev(v_new, torch.bfloat16, "v_new"),
                                      _dev(new_slots, torch.int32, "new_slots"), _dev(k_pool, torch.bfloat16, "k_pool"),
                                      _dev(v_pool, torch.bfloat16, "v_pool"), k_pool.shape[0],
                                      _dev(o, torch.bfloat16, "o"), _dev(ws, None, "ws"), ws_bytes, _stream(stream))
    _check(st, "rx_decode_cascade_append")


def rx_decode_run(cfg: AttnCfg, rtt, rec, rec_off, batches, max_seqs, shared_len: int, qs, ks, vs, k_pool, v_pool,
                  outs, ws, with_stable=True, stream=None, tp=None):
    """A run of decode steps in one C call (include/rx.h rx_decode_run): step k = one
    rx_decode_cascade_append / rx_decode_append over the records rec[rec_off[k]:] ([new slots |
    seq_lens | rows | stable lens], batches[k] int32 words each), q / k_new / v_new / o = qs[k] /
    ks[k] / vs[k] / outs[k] (CUDA bf16 tensors).  tp = (h_q_total, head_offset): fused-gather TP
    steps, outs[k] = the list of every rank's destination address (int) for step k."""
    import numpy as np
    import torch
    n = len(batches)
    for name, lst in (("q", qs), ("k_new", ks), ("v_new", vs)) + ((("o", outs),) if tp is None else ()):
        if len(lst) != n:
            raise ValueError(f"rx_decode_run: {name} needs {n} tensors")
        for t in lst:
            _dev(t, torch.bfloat16, name)
    b = np.ascontiguousarray(batches, dtype=np.int32)
    m = np.ascontiguousarray(max_seqs, dtype=np.int32)
    off = np.ascontiguousarray(rec_off, dtype=np.int64)
    ptrs = [(C.c_void_p * max(1, n))(*[t.data_ptr() for t in lst]) for lst in (qs, ks, vs)]
    if tp is None:
        optr, world, hq_total, head_off = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in outs]), 0, 0, 0
    else:
        if len(outs) != n or len({len(o) for o in outs}) > 1:
            raise ValueError("rx_decode_run: tp outs needs n lists of equal length")
        world = len(outs[0]) if n else 1
        flat = [int(a) for o in outs for a in o]
        optr = (C.c_void_p * max(1, len(flat)))(*flat)
        hq_total, head_off = int(tp[0]), int(tp[1])
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_decode_run(C.byref(cfg), n, b.ctypes.data_as(P32), m.ctypes.data_as(P32), shared_len,
                           _dev(rtt, torch.int32, "rtt"), rtt.shape[1], _dev(rec, torch.int32, "rec"),
                           off.ctypes.data_as(P64), 1 if with_stable else 0, ptrs[0], ptrs[1], ptrs[2],
                           _dev(k_pool, torch.bfloat16, "k_pool"), _dev(v_pool, torch.bfloat16, "v_pool"),
                           k_pool.shape[0], optr, world, hq_total, head_off, _dev(ws, None, "ws"), ws_bytes,
                           _stream(stream))
    _check(st, "rx_decode_run")


def tp_out(dests, h_q_total: int, head_offset: int):
    """rx_tp_out for rx_decode_append_tp: dests = device addresses (ints) of every rank's gathered
    output buffer [batch, h_q_total, head_dim] bf16 for this call, in rank order."""
    if not 1 <= len(dests) <= 8:
        raise ValueError("tp_out: 1..8 destinations")
    t = TpOut()
    for i, d in enumerate(dests):
        t.d_o[i] = int(d)
    t.world, t.h_q_total, t.head_offset = len(dests), h_q_total, head_offset
    return t


def rx_decode_append_tp(cfg: AttnCfg, rtt, rows, seq_lens, max_seq_len: int, shared_len: int, q, k_new, v_new,
                        new_slots, k_pool, v_pool, out, ws=None, stream=None, stable_lens=None):
    """TP decode step whose epilogue stores the output rows into every rank's gathered buffer
    (include/rx.h rx_decode_append_tp); `out` from tp_out()."""
    import torch
    batch = seq_lens.shape[0]
    ws_bytes = ws.numel() * ws.element_size() if ws is not None else 0
    st = lib.rx_decode_append_tp(C.byref(cfg), batch, _dev(rtt, torch.int32, "rtt"), rtt.shape[1],
                                 _dev(rows, torch.int32, "rows"), _dev(seq_lens, torch.int32, "seq_lens"),
                                 _dev(stable_lens, torch.int32, "stable_lens"), max_seq_len, shared_len,
                                 _dev(q, torch.bfloat16, "q"),
                                 _dev(k_new, torch.bfloat16, "k_new"), _dev(v_new, torch.bfloat16, "v_new"),
                                 _dev(new_slots, torch.int32, "new_slots"), _dev(k_pool, torch.bfloat16, "k_pool"),
                                 _dev(v_pool, torch.bfloat16, "v_pool"), k_pool.shape[0], C.byref(out),
                                 _dev(ws, None, "ws"), ws_bytes, _stream(stream))
    _check(st, "rx_decode_append_tp")


def rx_copy_h2d(dst, src_pinned, stream=None):
    """dst (CUDA tensor) <- src_pinned (pinned CPU tensor, same byte size), copied by an SM kernel."""
    import torch
    if not src_pinned.is_pinned():
        raise ValueError("rx_copy_h2d: the source must be pinned host memory")
    nb = src_pinned.numel() * src_pinned.element_size()
    if dst.numel() * dst.element_size() != nb:
        raise ValueError("rx_copy_h2d: size mismatch")
    _check(lib.rx_copy_h2d(_dev(dst, None, "dst"), C.c_void_p(src_pinned.data_ptr()), nb, _stream(stream)),
           "rx_copy_h2d")


def rx_last_launch_count() -> int:
    return lib.rx_last_launch_count()
