"""Fake tensor parallelism on one GPU: the P head shards of a
TP run, executed one after another on the same device, with exactly the
local shapes a P-GPU run uses.

* every shard's radix-tree trace is identical ("the tree
  operations are the same") and equals the 1-GPU trace;
* the shards' outputs, reassembled in global head order, match the 1-GPU run
  within the attention tolerance (different local shapes may change the
  split-KV partition, hence summation order, so not bitwise);
* the reassembled outputs match the fp64 ORACLE on every row within the
  north-star tolerance (max-abs 2e-2, mean-abs 2e-3).
"""
import types

import numpy as np
import pytest
import torch

from rxgen import workloads

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2312_07104_b200.engine import Engine, plan_and_bank


def _run(wl, rank=0, size=1):
    _, bank = plan_and_bank(wl, "cuda", tp_rank=rank, tp_size=size)
    e = Engine(wl, "cuda", tp_rank=rank, tp_size=size, record=True, keep_outputs=True)
    e.run_workload(bank)
    torch.cuda.synchronize()
    return e


@pytest.mark.parametrize("make,P", [
    (lambda: workloads.c5(n_req=6, prefix=600, question=40, decode=5, num_slots=8192), 2),
    (lambda: workloads.c5(n_req=6, prefix=600, question=40, decode=5, num_slots=8192), 8),
    (lambda: workloads.c3(sessions=4, turns=2, in_lo=30, in_hi=90, out_lo=4, out_hi=9, num_slots=8192), 8),
    (lambda: workloads.c1(), 4),
])
def test_fake_tp_matches_single_gpu(make, P):
    wl = make()
    full = _run(wl)
    shards = [_run(wl, r, P) for r in range(P)]
    for s in shards:
        assert s.trace == full.trace
    worst = 0.0
    for ci, (kind, o_full, _) in enumerate(full.outputs):
        parts = [s.outputs[ci][1] for s in shards]
        assert all(s.outputs[ci][0] == kind for s in shards)
        o_tp = torch.cat(parts, dim=1)                     # rank-major = global head order
        assert o_tp.shape == o_full.shape
        err = (o_tp.float() - o_full.float()).abs().max().item()
        worst = max(worst, err)
    assert worst <= 2e-2, worst
    # the re-assembled TP output against the oracle, every row (tests/test_gpu_engine.py::_compare)
    from test_gpu_engine import _compare, _all_ext, _all_dec
    tp = types.SimpleNamespace(outputs=[(kind, torch.cat([s.outputs[ci][1] for s in shards], dim=1), meta)
                                        for ci, (kind, _, meta) in enumerate(full.outputs)])
    oe = _compare(tp, wl, _all_ext, _all_dec)
    assert oe.trace == full.trace


@pytest.mark.parametrize("fused", [True, False])
def test_chunked_overlapped_gather_world1_nccl(fused):
    """The TP extend path with the output all-gather split into request blocks and overlapped with
    the next block's compute (NCCL async, one-rank group on this GPU): outputs are bit-identical to
    the unchunked call (blocks never split a request; each request's math is unchanged).  fused:
    decode steps through tp.FusedGather (rx_decode_append_tp: the epilogue stores into the gathered
    buffer, one barrier per decode run), else one NCCL all-gather per decode call."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2312_07104_b200.tp import make_gather
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    wl = workloads.c5(n_req=12, prefix=600, question=40, decode=3, num_slots=16384, ragged=True)
    ref = _run(wl)
    _, bank = plan_and_bank(wl, "cuda")
    g = make_gather(fused=fused)
    assert type(g).__name__ == ("FusedGather" if fused else "Gather")
    e = Engine(wl, "cuda", record=True, keep_outputs=True, gather=g)
    e.gather_chunk_rows = 100                       # several blocks for the 12 x U[64,256]-row extend
    assert e._gather_chunks(np.array([150] * 12)) is not None
    e.run_workload(bank)
    torch.cuda.synchronize()
    assert e.trace == ref.trace
    for (k1, o1, _), (k2, o2, _) in zip(ref.outputs, e.outputs):
        assert k1 == k2
        assert torch.equal(o1, o2.reshape(o1.shape))
    if fused:
        assert g.seq > 0                            # decode runs ended with their barriers
        g.close()
    dist.destroy_process_group()
