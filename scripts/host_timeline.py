"""Host timeline of one engine pass (dev tool): wall-clock start/end of the engine's phases (tree
work, staging, launches), relative to the pass start, after warm-up passes; plus the device span.

    python scripts/host_timeline.py C5
"""
import functools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from bench import make_workload
from paper_2312_07104_b200 import engine as E
from paper_2312_07104_b200.engine import Engine, plan_and_bank

LOG = []
DEPTH = [0]
METHODS = ["run_batch", "_reqs", "_match", "_run_matched", "_alloc", "_extend", "_extend_launch", "_finish_many",
           "_decode_loop_native", "_decode_launch", "_decode_phase", "_output_loop_py", "_upload", "_pinned"]


def wrap(name, fn):
    @functools.wraps(fn)
    def w(*a, **k):
        t0 = time.perf_counter()
        DEPTH[0] += 1
        try:
            return fn(*a, **k)
        finally:
            DEPTH[0] -= 1
            LOG.append((DEPTH[0], name, t0, time.perf_counter()))
    return w


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    wl = make_workload(name)
    plan, bank = plan_and_bank(wl, dev)
    eng = Engine(wl, dev)
    for _ in range(3):
        eng.reset()
        eng.run_workload(bank)
    for m in METHODS:
        if hasattr(Engine, m):
            setattr(Engine, m, wrap(m, getattr(Engine, m)))
    torch.cuda.synchronize()
    LOG.clear()
    eng.reset()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    t0 = time.perf_counter()
    s.record()
    eng.run_workload(bank)
    t1 = time.perf_counter()
    e.record()
    torch.cuda.synchronize()
    print(f"{name}: host {1e3 * (t1 - t0):.2f} ms, device span {s.elapsed_time(e):.2f} ms")
    agg = {}
    for d, n, a, b in LOG:
        x = agg.setdefault(n, [0, 0.0])
        x[0] += 1
        x[1] += b - a
    for n, (c, tt) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"  {n:22s} x{c:5d}  {1e3 * tt:8.2f} ms")
    if len(LOG) < 400:
        for d, n, a, b in sorted(LOG, key=lambda x: x[2]):
            print(f"  {'  ' * d}{n:22s} {1e3 * (a - t0):8.3f} .. {1e3 * (b - t0):8.3f} ms")


if __name__ == "__main__":
    main()
