"""Timeline of extend-kernel CTA 0 (development tool; needs RX_EXT_TRACE=1).

    RX_EXT_TRACE=1 python scripts/ext_trace.py --h 32 8 128 --batch 256 --prefix 0 --ext 384
Codes: 1 Q issued, 2 K tile issued, 3 V tile issued, 4 S issued, 5 P seen by MMA, 6 PV issued,
       7 softmax has S, 8 softmax P done, 9 epilogue start, 10 epilogue end.
"""
import argparse
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2312_07104_b200 as rx
from paper_2312_07104_b200._lib import lib

NAMES = {1: "Q", 2: "K", 3: "V", 4: "S", 5: "Pseen", 6: "PV", 7: "smS", 8: "smP", 9: "epi0", 10: "epi1"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, nargs=3, default=[32, 8, 128])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--prefix", type=int, default=0)
    ap.add_argument("--ext", type=int, default=384)
    a = ap.parse_args()
    h_q, h_kv, hd = a.h
    B, P, E = a.batch, a.prefix, a.ext
    dev = "cuda"
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    S = B * (P + E) + 16
    kp = torch.randn((S, h_kv, hd), device=dev).to(torch.bfloat16)
    vp = torch.randn_like(kp)
    rtt = (torch.arange(B * (P + E), dtype=torch.int32, device=dev) + 1).view(B, P + E)
    N = B * E
    q = torch.randn((N, h_q, hd), device=dev).to(torch.bfloat16)
    kn = torch.randn((N, h_kv, hd), device=dev).to(torch.bfloat16)
    vn = torch.randn_like(kn)
    o = torch.empty_like(q)
    pre = torch.full((B,), P, dtype=torch.int32, device=dev)
    ext = torch.full((B,), E, dtype=torch.int32, device=dev)
    ind = torch.arange(B + 1, dtype=torch.int32, device=dev) * E
    f = lib.rx_debug_ext_trace
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int]
    for _ in range(2):
        rx.rx_extend(cfg, rtt, None, pre, ext, ind, N, E, P, q, kn, vn, kp, vp, o)
        torch.cuda.synchronize()
        f(None, 0)
    rx.rx_extend(cfg, rtt, None, pre, ext, ind, N, E, P, q, kn, vn, kp, vp, o)
    buf = (C.c_ulonglong * 8192)()
    n = f(buf, 8192)
    recs = np.frombuffer(buf, dtype=np.uint64)[:n]
    code = (recs >> np.uint64(56)).astype(int)
    item = ((recs >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(int)
    clk = (recs & np.uint64(0xFFFFFFFF)).astype(np.int64)
    clk = (clk - clk.min()) % (1 << 32)
    order = np.argsort(clk, kind="stable")
    print(f"{n} records; span {clk.max()} cycles")
    last = {}
    for i in order[:400]:
        c, it, t = code[i], item[i], clk[i]
        dt = t - last.get(c, t)
        last[c] = t
        print(f"{t:10d}  {NAMES.get(c, c):6s} #{it:<5d} (+{dt} since prev {NAMES.get(c, c)})")
    # per-code average interval
    for c in sorted(set(code)):
        ts = np.sort(clk[code == c])
        if len(ts) > 2:
            print(f"{NAMES.get(c, c):6s}: {len(ts)} events, mean interval {np.diff(ts).mean():.0f} cycles")


if __name__ == "__main__":
    main()
