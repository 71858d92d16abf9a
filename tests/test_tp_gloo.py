"""Multi-process (world_size 2, gloo, CPU) coverage of the TP host path:
head sharding covers every head exactly once, every rank's replicated tree
ends identical ("the tree operations are the same"), and the
all-gather reassembles head shards in global head order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2312_07104_b200.engine import Engine, shard_heads
        from paper_2312_07104_b200.tp import make_gather, check_replicated, tree_digest
        from rxgen import workloads
        wl = workloads.c5(n_req=6, prefix=200, question=17, decode=4, num_slots=4096)
        e = Engine(wl, plan_only=True, tp_rank=rank, tp_size=world)
        e.run_workload()
        ok_tree = check_replicated(e.cache)
        # gather: each rank holds o for its own heads; global head index h in every element
        qh, kvh = shard_heads(64, 8, rank, world)
        n, hd = 5, 4
        o_local = torch.tensor(qh, dtype=torch.float32).view(1, -1, 1).expand(n, -1, hd).contiguous()
        full = make_gather()(o_local).reshape(n, -1, hd)
        ok_gather = torch.equal(full[0, :, 0], torch.arange(64, dtype=torch.float32))
        q.put((rank, ok_tree, ok_gather, tree_digest(e.cache), qh, kvh))
        dist.destroy_process_group()
    except Exception as ex:  # surface errors to the parent
        q.put((rank, "error", repr(ex)))


def test_tp_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    res.sort(key=lambda r: r[0])
    for r in res:
        assert r[1] != "error", r
        assert r[1] is True and r[2] is True, r
    assert res[0][3] == res[1][3]
    assert res[0][4] + res[1][4] == list(range(64))
    assert res[0][5] == [0, 1, 2, 3] and res[1][5] == [4, 5, 6, 7]
