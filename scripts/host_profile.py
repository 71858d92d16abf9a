"""Host-side profile of one engine pass (dev tool): wall time of the pass, device time (events), and
the top host functions by cumulative time (cProfile), after warm-up passes.

    python scripts/host_profile.py C5
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from bench import make_workload
from paper_2312_07104_b200.engine import Engine, plan_and_bank


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
    torch.cuda.synchronize()
    for _ in range(3):
        eng.reset()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        s.record()
        eng.run_workload(bank)
        t1 = time.perf_counter()
        e.record()
        torch.cuda.synchronize()
        print(f"{name}: host enqueue {1e3 * (t1 - t0):.2f} ms, device span {s.elapsed_time(e):.2f} ms")
    eng.reset()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    eng.run_workload(bank)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
