"""Tensor parallelism over KV heads (§3).

"For tensor parallelism, each GPU maintains a sharded KV cache. There is no
need for additional synchronization because the tree operations are the
same."  So:

* every rank runs its own rx_cache on the identical op sequence (slot indices
  agree with no communication; ``tree_digest`` lets a debug run all-reduce a
  hash of the tree to prove it);
* rank r owns q heads [r*H_q/P, (r+1)*H_q/P) and the kv heads they read, i.e.
  its slice of the pool (``engine.shard_heads``);
* the only exchange is ONE all-gather of the bf16 attention output per call.
  Decode steps (thousands per C3 step): ``FusedGather`` (default on a CUDA
  group) — the attention epilogue stores every output row into every rank's
  IPC-mapped buffer (rx_decode_append_tp), one flag barrier per decode run;
  no collective per step.  Otherwise NCCL ``all_gather_into_tensor``
  (``Gather``), or ``P2PGather`` (librx rx_tp_allgather: one kernel stores the
  shard into every peer's buffer and synchronises with flags; RX_TP_P2P=1);
  extend calls use NCCL (chunked, overlapped with the next block's compute).
"""
from __future__ import annotations

import hashlib
import json

import torch
import torch.distributed as dist


def _map_peers(lib, buf, world, rank, group):
    """Export this rank's buffer (IPC handle + its offset inside the handle's allocation) and map
    every peer's: (opened base pointers to close later, [device address of rank r's buffer])."""
    import ctypes as C
    h = (C.c_uint8 * 64)()
    st = lib.rx_tp_ipc_handle(C.c_void_p(buf.data_ptr()), C.cast(h, C.c_void_p))
    off = lib.rx_tp_ipc_offset(C.c_void_p(buf.data_ptr()))
    if st != 0 or off < 0:
        raise RuntimeError(f"rx_tp_ipc_handle / rx_tp_ipc_offset: {st} / {off}")
    handles = [None] * world
    dist.all_gather_object(handles, (bytes(h), int(off)), group=group)
    opened, ptrs = [], []
    for r, (hb, o) in enumerate(handles):
        if r == rank:
            ptrs.append(buf.data_ptr())
            continue
        p = C.c_void_p()
        st = lib.rx_tp_ipc_open(C.cast((C.c_uint8 * 64).from_buffer_copy(hb), C.c_void_p), C.byref(p))
        if st != 0:
            raise RuntimeError(f"rx_tp_ipc_open(rank {r}): {st}")
        opened.append(p)
        ptrs.append(p.value + o)
    return opened, ptrs


class Gather:
    """gather(o_local [N, hq_local, hd]) -> o [N, P, hq_local, hd].

    The result is a strided VIEW of the rank-major all-gather buffer [P, N,
    hq_local, hd]: global q head = rank * hq_local + local head.  No permute
    copy is made (callers that need a dense [N, H_q, hd] reshape it).

    Chunked form for large calls (a C5 suffix extend gathers
    268 MB): ``alloc`` the buffer, ``start`` an asynchronous all-gather of
    each finished row block while the next block computes (NCCL's stream waits
    only for the work enqueued before the call), ``finish`` joins them."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.tensor_api = dist.get_backend(group) == "nccl"

    def __call__(self, o_local: torch.Tensor) -> torch.Tensor:
        o_local = o_local.contiguous()
        out = torch.empty((self.world,) + tuple(o_local.shape), dtype=o_local.dtype, device=o_local.device)
        if self.tensor_api:
            dist.all_gather_into_tensor(out, o_local, group=self.group)
        else:
            dist.all_gather(list(out.unbind(0)), o_local, group=self.group)
        return out.permute(1, 0, 2, 3)

    def alloc(self, n, hq_local, hd, dtype, device):
        return torch.empty((self.world, n, hq_local, hd), dtype=dtype, device=device)

    def start(self, o_part: torch.Tensor, out: torch.Tensor, r0: int, r1: int):
        """all-gather rows [r0, r1) of every rank into out[:, r0:r1] (async)."""
        return dist.all_gather([out[r, r0:r1] for r in range(self.world)], o_part.contiguous(), group=self.group,
                               async_op=True)

    @staticmethod
    def finish(handles, out):
        for h in handles:
            h.wait()
        return out.permute(1, 0, 2, 3)


class P2PGather:
    """gather(o_local) over peer memory (include/rx.h section 3): every rank holds one zero-filled
    IPC buffer of rx_tp_buffer_bytes(world, cap); handles are exchanged once through the process
    group; each call is one rx_tp_allgather kernel on the current stream plus one device copy of the
    gathered [P, bytes] slot into a fresh tensor (so the result outlives the two-slot ring).  Calls
    whose shard exceeds `cap` bytes, and the chunked extend gathers (alloc / start / finish), go
    through NCCL (``Gather``)."""

    def __init__(self, cap_bytes=8 << 20, group=None, device=None):
        import ctypes as C
        from ._lib import lib
        self._lib, self._C = lib, C
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cap = (int(cap_bytes) + 15) // 16 * 16
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buf = torch.zeros(int(lib.rx_tp_buffer_bytes(self.world, self.cap)), dtype=torch.uint8, device=dev)
        self._opened, ptrs = _map_peers(lib, self.buf, self.world, self.rank, group)
        self.peers = (C.c_void_p * self.world)(*ptrs)
        self.seq = 0
        self.fallback = Gather(group)
        dist.barrier(group=group)              # every rank mapped every buffer before the first call

    def __call__(self, o_local: torch.Tensor) -> torch.Tensor:
        o_local = o_local.contiguous()
        n = o_local.numel() * o_local.element_size()
        if n > self.cap or n % 16:
            return self.fallback(o_local)
        self.seq += 1
        C = self._C
        st = self._lib.rx_tp_allgather(C.c_void_p(o_local.data_ptr()), n, self.peers, self.world, self.rank,
                                       self.cap, self.seq, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        if st != 0:
            raise RuntimeError(f"rx_tp_allgather: {st}")
        base = 256 + (self.seq & 1) * self.world * self.cap
        slot = self.buf[base:base + self.world * self.cap].view(self.world, self.cap)[:, :n]
        out = torch.empty((self.world,) + tuple(o_local.shape), dtype=o_local.dtype, device=o_local.device)
        out.view(self.world, -1).view(torch.uint8).copy_(slot)
        return out.permute(1, 0, 2, 3)

    # chunked, overlapped extend gathers: NCCL
    def alloc(self, n, hq_local, hd, dtype, device):
        return self.fallback.alloc(n, hq_local, hd, dtype, device)

    def start(self, o_part, out, r0, r1):
        return self.fallback.start(o_part, out, r0, r1)

    @staticmethod
    def finish(handles, out):
        return Gather.finish(handles, out)

    def close(self):
        for p in self._opened:
            self._lib.rx_tp_ipc_close(p)
        self._opened = []


class FusedGather:
    """Decode outputs gathered by the attention epilogue itself (include/rx.h rx_decode_append_tp):
    the kernel that produces a final output row stores it into EVERY rank's gathered buffer over
    peer memory, so a decode step has no collective, no extra kernel and no copy.

    Every rank holds one IPC buffer: [256-byte barrier header | region 0 | region 1] (regions of
    ``region_bytes``, holding gathered rows [h_q_total, head_dim] bf16); every rank maps every
    peer's buffer.
    A decode run (the calls of one engine decode launch) takes consecutive rows of region
    (run & 1) — the same rows on every rank, because every rank issues the identical call
    sequence — and ends with ONE rx_tp_allgather(bytes = 0) barrier: its flags publish "my stores
    of this run are done" and wait for every peer's, after which this rank's region holds the
    whole gathered output of the run.  A peer writes region (run & 1) again only in run + 2,
    i.e. after this rank's barrier of run + 1, which the engine issues only once its readers of
    run (the host sink's copies) are done.  Extend calls (few, large) use NCCL (``Gather``)."""

    fused = True

    def __init__(self, region_bytes=256 << 20, group=None, device=None, fallback=None, host_barrier=False):
        import ctypes as C
        from ._lib import lib
        self._lib, self._C = lib, C
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.region_bytes = (int(region_bytes) + 255) // 256 * 256
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buf = torch.zeros(256 + 2 * self.region_bytes, dtype=torch.uint8, device=dev)
        self._opened, ptrs = _map_peers(lib, self.buf, self.world, self.rank, group)
        self.ptrs = ptrs
        self.peers = (C.c_void_p * self.world)(*ptrs)
        self.run = 0
        self.used = 0
        self.seq = 0
        self.fallback = fallback if fallback is not None else Gather(group)
        # host_barrier (tests with several ranks on ONE device): end a run by synchronising this
        # rank's device and a process-group barrier instead of the device flag barrier — ranks that
        # time-share one GPU must not spin in a kernel on work of a context that is not running
        # (one process per GPU, the deployment, uses the device barrier)
        self.host_barrier = host_barrier
        dist.barrier(group=group)              # every rank mapped every buffer before the first call

    def begin_run(self):
        self.run += 1
        self.used = 0

    def fits(self, rows, h_q_total, head_dim):
        return self.used + (rows * h_q_total * head_dim * 2 + 255) // 256 * 256 <= self.region_bytes

    def take(self, rows, h_q_total, head_dim):
        """(destination addresses on every rank, this rank's view [rows, h_q_total, head_dim]) of
        the next gathered block of the current run."""
        n = rows * h_q_total * head_dim * 2
        if not self.fits(rows, h_q_total, head_dim):
            raise RuntimeError(f"FusedGather: run exceeds {self.region_bytes} bytes (end the run first)")
        off = 256 + (self.run & 1) * self.region_bytes + self.used
        self.used += (n + 255) // 256 * 256
        view = self.buf[off:off + n].view(torch.bfloat16).view(rows, h_q_total, head_dim)
        return [p + off for p in self.ptrs], view

    def end_run(self):
        """The run's barrier on the current stream (every rank's stores of the run are visible)."""
        self.seq += 1
        if self.host_barrier:
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
            return
        C = self._C
        st = self._lib.rx_tp_allgather(None, 0, self.peers, self.world, self.rank, 16, self.seq,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream))
        if st != 0:
            raise RuntimeError(f"rx_tp_allgather (barrier): {st}")

    # extend calls: NCCL
    def __call__(self, o_local):
        return self.fallback(o_local)

    def alloc(self, n, hq_local, hd, dtype, device):
        return self.fallback.alloc(n, hq_local, hd, dtype, device)

    def start(self, o_part, out, r0, r1):
        return self.fallback.start(o_part, out, r0, r1)

    @staticmethod
    def finish(handles, out):
        return Gather.finish(handles, out)

    def close(self):
        for p in self._opened:
            self._lib.rx_tp_ipc_close(p)
        self._opened = []


def make_gather(group=None, p2p=None, fused=None):
    """The TP output gather: NCCL (Gather) by default; the peer-memory P2PGather when p2p=True or
    RX_TP_P2P=1 on a CUDA (NCCL) group.  (Measured on one rank: NCCL's gather costs 7 us of device
    time per call, P2PGather 21 us — its kernel + copy + launch — so P2P is opt-in until a fused
    epilogue store removes the separate copy.)"""
    import os
    if p2p is None:
        p2p = os.environ.get("RX_TP_P2P", "0") == "1"
    if fused is None:
        fused = os.environ.get("RX_TP_FUSED", "1") == "1"
    nccl = dist.get_backend(group) == "nccl"
    if fused and nccl:
        return FusedGather(group=group)
    if p2p and nccl:
        return P2PGather(group=group)
    return Gather(group)


def tree_digest(cache) -> str:
    """sha256 of the tree's deterministic pre-order dump (ids, tokens, slots, refs, stamps)."""
    return hashlib.sha256(json.dumps(cache.rx_dump_json(), separators=(",", ":")).encode()).hexdigest()


def check_replicated(cache, group=None) -> bool:
    """All ranks hold the identical tree (debug mode of SURVEY §8(e))."""
    d = torch.tensor(list(bytes.fromhex(tree_digest(cache))[:8]), dtype=torch.int64)
    lo, hi = d.clone(), d.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return bool(torch.equal(lo, hi))
