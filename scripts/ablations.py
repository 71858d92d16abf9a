"""GPU ablations of the paper's §6, each a whole pass of the hot path, CUDA events,
L2 flushed, median of --steps after --warmup.

  sched: the MIX queue (interleaved few-shot groups that do not all fit the pool) under each
         rx_schedule policy ("FCFS Schedule" / "Random Schedule" vs cache-aware LSPF,
         P:214-219).  Same requests and outputs; the hit rate decides the extend work.
  fsm:   JSON decoding under a regex: compressed FSM (jump forward, one pass per sampled
         token + its forced edge) vs token-by-token decoding.  Same output text.

    python scripts/ablations.py [sched|fsm|all] [--steps 5] [--warmup 3]

One JSON line per variant: hit rate (cached prompt tokens / prompt tokens), tokens computed,
forward passes, ms per pass, served tokens/s = (prompt + output tokens) / time (same numerator for
every variant of an ablation).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2312_07104_b200.engine import Engine, plan_and_bank
from rxgen import workloads


def _time(wl, dev, flush, steps, warmup, policy="lspf"):
    plan, bank = plan_and_bank(wl, dev, policy=policy)
    eng = Engine(wl, dev, policy=policy)
    for _ in range(warmup):
        eng.reset()
        eng.run_workload(bank)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
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
    return {"hit_rate": st["cached_prompt_tokens"] / st["prompt_tokens"],
            "extend_tokens": st["extend_tokens"], "output_tokens": st["output_tokens"],
            "passes": len(plan.calls), "extend_calls": sum(1 for c in plan.calls if c.kind == "extend"),
            "ms_per_pass": ms, "served_tokens_per_s": (st["prompt_tokens"] + st["output_tokens"]) / (ms / 1000.0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="?", default="all", choices=["sched", "fsm", "all"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
    if a.which in ("sched", "all"):
        for policy in ("lspf", "fcfs", "random"):
            r = _time(workloads.mix(), dev, flush, a.steps, a.warmup, policy)
            print(json.dumps({"ablation": "sched", "workload": "MIX (4 groups x 16, 1024-token prefixes, pool 2600)",
                              "policy": policy, **r}))
    if a.which in ("fsm", "all"):
        for n_req, prefix in ((64, 512), (256, 1024)):
            for comp in (True, False):
                r = _time(workloads.json_decode(n_req=n_req, prefix=prefix, compressed=comp, num_slots=1 << 18), dev,
                          flush, a.steps, a.warmup)
                # output tokens include the start edge prefilled with the prompt (compressed mode)
                print(json.dumps({"ablation": "fsm", "workload": f"JSON ({n_req} req, {prefix}-token shared "
                                  "instruction, character-profile regex)", "compressed": comp, **r}))


if __name__ == "__main__":
    main()
