"""Per-kernel breakdown of shared-prefix (cascade) decode steps (dev tool, not the bench contract).

Runs `--steps` back-to-back rx_decode_cascade_append calls (the in-bench chain: programmatic
dependent launches, no L2 flush between steps) on the C5 or C2 shape and reports, from a
torch.profiler (CUPTI) trace, each kernel's mean device duration and the mean step span.

    python scripts/cascade_breakdown.py --shape C5 --steps 32
"""
import argparse
import math
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2312_07104_b200 as rx

SHAPES = {"C5": ((64, 8, 128), 128, 8320, 8192), "C2": ((32, 32, 128), 64, 1700, 1536),
          # C4 (tree of thought on a 2k root, G = 1): level-1 / level-2 / level-3 decode batches
          "C4a": ((32, 32, 128), 4, 2160, 2048), "C4b": ((32, 32, 128), 16, 2200, 2048),
          "C4c": ((32, 32, 128), 64, 2240, 2048)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", choices=sorted(SHAPES), default="C5")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--per-request", action="store_true", help="time rx_decode_append instead")
    ap.add_argument("--no-stable", action="store_true", help="no stable region (wait before any read)")
    a = ap.parse_args()
    (h_q, h_kv, hd), B, L0, P = SHAPES[a.shape]
    dev = "cuda"
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    g = torch.Generator(device=dev).manual_seed(0)
    Lmax = L0 + a.steps
    S = P + B * (Lmax - P) + 16
    kp = torch.randn((S, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
    vp = torch.randn_like(kp)
    rtt = torch.zeros((B, Lmax), dtype=torch.int32, device=dev)
    rtt[:, :P] = torch.arange(1, P + 1, dtype=torch.int32, device=dev)
    own = torch.arange(P + 1, P + 1 + B * (Lmax - P), dtype=torch.int32, device=dev).view(B, Lmax - P)
    rtt[:, P:L0 - 1] = own[:, :L0 - 1 - P]
    q = torch.randn((a.steps, B, h_q, hd), device=dev, generator=g).to(torch.bfloat16)
    kn = torch.randn((a.steps, B, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
    vn = torch.randn_like(kn)
    o = torch.empty((B, h_q, hd), dtype=torch.bfloat16, device=dev)
    stable = None if a.no_stable else torch.full((B,), L0 - 1, dtype=torch.int32, device=dev)
    lens = [torch.full((B,), L0 + t, dtype=torch.int32, device=dev) for t in range(a.steps)]
    news = [own[:, L0 - 1 - P + t].contiguous() for t in range(a.steps)]
    wsb = max(rx.rx_decode_cascade_workspace_bytes(cfg, B, Lmax, P), rx.rx_decode_workspace_bytes(cfg, B, Lmax))
    ws = torch.zeros(wsb + 1, dtype=torch.uint8, device=dev)

    def chain():
        for t in range(a.steps):
            if a.per_request:
                rx.rx_decode_append(cfg, rtt, None, lens[t], L0 + t, q[t], kn[t], vn[t], news[t], kp, vp, o, ws,
                                    stable_lens=stable)
            else:
                rx.rx_decode_cascade_append(cfg, rtt, None, lens[t], L0 + t, P, q[t], kn[t], vn[t], news[t], kp, vp,
                                            o, ws, stable_lens=stable)

    chain()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    chain()
    e.record()
    torch.cuda.synchronize()
    span = s.elapsed_time(e) * 1e3 / a.steps
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        chain()
        torch.cuda.synchronize()
    dur = defaultdict(list)
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            dur[ev.name[:60]].append(ev.device_time)
    print(f"{a.shape} {'per-request' if a.per_request else 'cascade'} B={B} L={L0}..{Lmax} shared={P}: "
          f"{span:.1f} us per step (events, {a.steps} chained steps)")
    for k, v in sorted(dur.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {sum(v)/a.steps:8.1f} us/step  {sum(v)/len(v):8.1f} us x {len(v)/a.steps:.0f}  {k}")


if __name__ == "__main__":
    main()
