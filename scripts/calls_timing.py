"""Per-call device times of one workload pass (dev tool): every extend call with its shape and
TFLOP/s, and decode calls aggregated per batch phase.  CUDA events on the launching stream, L2
flushed before the pass, after warm-up passes.

    python scripts/calls_timing.py [C3|C5|C2|JSON|MIX] [--warmup 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from bench import make_workload
from paper_2312_07104_b200.engine import Engine, plan_and_bank
from rxgen import workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", default="C3", nargs="?")
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    extra = {"JSON": workloads.json_decode, "MIX": workloads.mix}
    wl = extra[a.workload]() if a.workload in extra else make_workload(a.workload)
    plan, bank = plan_and_bank(wl, dev)
    eng = Engine(wl, dev)
    for _ in range(a.warmup):
        eng.reset()
        eng.run_workload(bank)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
    flush.fill_(1)
    torch.cuda.synchronize()
    eng.reset()
    eng.enable_timing(True)
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    eng.run_workload(bank)
    e.record()
    torch.cuda.synchronize()
    total = s.elapsed_time(e)
    ext_calls = [c for c in plan.calls if c.kind == "extend"]
    ei = 0
    dec_ms, dec_n, dec_bytes = 0.0, 0, 0.0
    kern_ms = 0.0
    prev_end = s
    for kind, ev0, ev1, work, nl, calls in eng.timer:
        ms = ev0.elapsed_time(ev1)
        kern_ms += ms
        if kind == "extend":
            print(f"  (gap before this extend: {prev_end.elapsed_time(ev0):.3f} ms)")
        prev_end = ev1
        if kind == "extend":
            meta = ext_calls[ei].meta
            ei += 1
            ext = np.array(meta["ext"])
            pre = np.array(meta.get("prefix", [0] * len(ext)))
            print(f"extend B={len(ext):4d} new={ext.sum():7d} (max {ext.max():5d}) prefix sum={pre.sum():9d} "
                  f"max={pre.max():6d}: {ms:8.3f} ms {work / ms / 1e9:7.1f} TFLOP/s launches={nl}")
        else:
            dec_ms += ms
            dec_n += calls
            dec_bytes += sum(eng.decode_bytes(w)[0] for w in work)
    if dec_n:
        print(f"decode: {dec_n} calls {dec_ms:.2f} ms {dec_bytes / dec_ms / 1e6:.1f} GB/s (algorithmic)")
    print(f"pass {total:.2f} ms, kernels (event-bracketed) {kern_ms:.2f} ms, gaps {total - kern_ms:.2f} ms")


if __name__ == "__main__":
    main()
