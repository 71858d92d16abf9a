"""Timeline of extend-kernel CTA 0 (development tool; needs RX_EXT_TRACE=1).

    RX_EXT_TRACE=1 python scripts/ext_trace.py --h 32 8 128 --batch 256 --prefix 0 --ext 384
Codes: 1 Q issued, 2 K tile issued, 3 V tile issued, 4 S issued, 5 P seen by MMA, 6 PV issued,
       7 softmax has S, 8 softmax P done, 9 epilogue start, 10 epilogue end, 11 K landed (seen by
       the MMA warp), 12 V landed, 13 S MMAs issued, 14 PV MMAs issued, 15 MMA warp waits for K.
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

NAMES = {1: "Q", 2: "K", 3: "V", 4: "S", 5: "Pseen", 6: "PV", 7: "smS", 8: "smP", 9: "epi0", 10: "epi1",
         11: "Kin", 12: "Vin", 13: "Smma", 14: "PVmma", 15: "Kwait"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h", type=int, nargs=3, default=[32, 8, 128])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--prefix", type=int, default=0)
    ap.add_argument("--ext", type=int, default=384)
    ap.add_argument("--tiles", type=int, nargs=2, default=None, help="print per-tile event times for tiles [a, b)")
    ap.add_argument("--log", type=int, nargs=2, default=None, help="time-ordered event log of tiles [a, b)")
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
    buf = (C.c_ulonglong * (16 * 1024))()
    f(buf, 16 * 1024)
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(16, 1024)
    t0 = t[t > 0].min()
    t = np.where(t > 0, t - t0, -1)
    for c in sorted(NAMES):
        v = np.sort(t[c][t[c] >= 0])
        if len(v) > 2:
            print(f"{NAMES[c]:6s}: {len(v)} events, mean interval {np.diff(v).mean():.0f} cycles, span {v[-1]}")
    # per-tile latencies (tile index g): S issue -> softmax has S -> P done -> PV issue
    S, smS, smP, PV = t[4], t[7], t[8], t[6]
    ok = (S >= 0) & (smS >= 0) & (smP >= 0) & (PV >= 0)
    if ok.any():
        print("tile: S->smS %.0f  smS->smP %.0f  smP->PV %.0f  (mean cycles over %d tiles)" % (
            (smS - S)[ok].mean(), (smP - smS)[ok].mean(), (PV - smP)[ok].mean(), ok.sum()))
    if a.tiles:
        codes = [2, 3, 11, 4, 7, 8, 5, 12, 6]
        print("tile " + " ".join(f"{NAMES[c]:>7s}" for c in codes) + "   (cycles since the tile's K issue)")
        for g in range(*a.tiles):
            z = t[2][g]
            print(f"{g:4d} " + " ".join(f"{(t[c][g] - z) if t[c][g] >= 0 else -1:7d}" for c in codes))
    if a.log:
        ev = [(t[c][g], NAMES[c], g) for g in range(*a.log) for c in NAMES if c not in (1, 9, 10) and t[c][g] >= 0]
        ev.sort()
        z = ev[0][0]
        for tt, n, g in ev:
            print(f"{tt - z:8d}  {n:6s} tile {g}")
    q, e0, e1 = t[1], t[9], t[10]
    ok = (e0 >= 0) & (e1 >= 0)
    if ok.any():
        print("item epilogue %.0f cycles (mean over %d items)" % ((e1 - e0)[ok].mean(), ok.sum()))


if __name__ == "__main__":
    main()
