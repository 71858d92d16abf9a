"""Tensor parallelism over KV heads (§3).

"For tensor parallelism, each GPU maintains a sharded KV cache. There is no
need for additional synchronization because the tree operations are the
same."  So:

* every rank runs its own rx_cache on the identical op sequence (slot indices
  agree with no communication; ``tree_digest`` lets a debug run all-reduce a
  hash of the tree to prove it);
* rank r owns q heads [r*H_q/P, (r+1)*H_q/P) and the kv heads they read, i.e.
  its slice of the pool (``engine.shard_heads``);
* the only exchange is ONE all_gather of the bf16 attention output per call,
  over NCCL on NVLink (torch.distributed), returned as a strided view — no
  permute copy.
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


def make_gather(group=None):
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
