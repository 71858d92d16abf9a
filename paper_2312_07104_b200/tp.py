"""Tensor parallelism over KV heads (§3).

"For tensor parallelism, each GPU maintains a sharded KV cache. There is no
need for additional synchronization because the tree operations are the
same."  So:

* every rank runs its own rx_cache on the identical op sequence (slot indices
  agree with no communication; ``tree_digest`` lets a debug run all-reduce a
  hash of the tree to prove it);
* rank r owns q heads [r*H_q/P, (r+1)*H_q/P) and the kv heads they read, i.e.
  its slice of the pool (``engine.shard_heads``);
* the only exchange is ONE all-gather of the bf16 attention output per call:
  NCCL ``all_gather_into_tensor`` (``Gather``, default), or ``P2PGather``
  (librx rx_tp_allgather: one kernel stores the shard into every peer's
  IPC-mapped buffer over NVLink and synchronises with flags; opt-in,
  RX_TP_P2P=1), with NCCL for the chunked, overlapped extend gathers.
"""
from __future__ import annotations

import hashlib
import json

import torch
import torch.distributed as dist


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
        h = (C.c_uint8 * 64)()
        st = lib.rx_tp_ipc_handle(C.c_void_p(self.buf.data_ptr()), C.cast(h, C.c_void_p))
        if st != 0:
            raise RuntimeError(f"rx_tp_ipc_handle: {st}")
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        self._opened = []
        ptrs = []
        for r, hb in enumerate(handles):
            if r == self.rank:
                ptrs.append(self.buf.data_ptr())
                continue
            p = C.c_void_p()
            hh = (C.c_uint8 * 64).from_buffer_copy(hb)
            st = lib.rx_tp_ipc_open(C.cast(hh, C.c_void_p), C.byref(p))
            if st != 0:
                raise RuntimeError(f"rx_tp_ipc_open(rank {r}): {st}")
            self._opened.append(p)
            ptrs.append(p.value)
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


def make_gather(group=None, p2p=None):
    """The TP output gather: NCCL (Gather) by default; the peer-memory P2PGather when p2p=True or
    RX_TP_P2P=1 on a CUDA (NCCL) group.  (Measured on one rank: NCCL's gather costs 7 us of device
    time per call, P2PGather 21 us — its kernel + copy + launch — so P2P is opt-in until a fused
    epilogue store removes the separate copy.)"""
    import os
    if p2p is None:
        p2p = os.environ.get("RX_TP_P2P", "0") == "1"
    if p2p and dist.get_backend(group) == "nccl":
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
