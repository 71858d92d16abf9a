"""Scheduling ablation on the GPU ("FCFS Schedule" / "Random Schedule" vs cache-aware LSPF,
P:214-219): the MIX queue (interleaved few-shot groups that do not all fit the pool) run through the
whole hot path under each rx_schedule policy.  Same requests, same outputs; what changes is how many
prompt tokens hit the cache and therefore how much extend work is done.

    python scripts/sched_ablation.py [--steps 5] [--warmup 3]

Prints one JSON line per policy: hit rate (cached prompt tokens / prompt tokens), extend and
decode tokens computed, ms per pass (CUDA events, L2 flushed), served tokens/s = (prompt + decode
tokens of the queue) / time, the same numerator for every policy.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2312_07104_b200.engine import Engine, plan_and_bank
from rxgen import workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
    for policy in ("lspf", "fcfs", "random"):
        wl = workloads.mix()
        plan, bank = plan_and_bank(wl, dev, policy=policy)
        eng = Engine(wl, dev, policy=policy)
        for _ in range(a.warmup):
            eng.reset()
            eng.run_workload(bank)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            eng.reset()
            s.record()
            eng.run_workload(bank)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        st = plan.stats
        ms = sorted(ts)[len(ts) // 2]
        served = st["prompt_tokens"] + st["decode_tokens"]
        print(json.dumps({"workload": "MIX (4 groups x 16, 1024-token prefixes, pool 2600)", "policy": policy,
                          "hit_rate": st["cached_prompt_tokens"] / st["prompt_tokens"],
                          "extend_tokens": st["extend_tokens"], "decode_tokens": st["decode_tokens"],
                          "waves": sum(1 for c in plan.calls if c.kind == "extend"),
                          "ms_per_pass": ms, "served_tokens_per_s": served / (ms / 1000.0)}))


if __name__ == "__main__":
    main()
