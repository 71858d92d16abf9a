"""Quick per-kernel timing on synthetic shapes (not the bench contract; a dev tool).

    python scripts/kbench.py decode --h 32 8 128 --batch 256 --seq 2048
    python scripts/kbench.py extend --h 64 8 128 --batch 128 --prefix 8192 --ext 128
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2312_07104_b200 as rx


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["decode", "extend", "store"])
    ap.add_argument("--h", type=int, nargs=3, default=[32, 8, 128])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--prefix", type=int, default=0)
    ap.add_argument("--ext", type=int, default=512)
    ap.add_argument("--shared-prefix", action="store_true")
    ap.add_argument("--scatter", action="store_true", help="fragmented (non-contiguous) slots")
    ap.add_argument("--ragged", action="store_true", help="extend: prefix U[P/2, 3P/2], ext U[2E/3, 4E/3] per request")
    ap.add_argument("--half", action="store_true", help="extend: scatter every other 384-token run of the prefix "
                    "(C3 history: contiguous inputs, interleaved decode outputs)")
    ap.add_argument("--cascade", type=int, default=0, help="decode: shared prefix length (cascade vs per-request)")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    h_q, h_kv, hd = a.h
    B = a.batch
    dev = "cuda"
    cfg = rx.attn_cfg(h_q, h_kv, hd, 1 / math.sqrt(hd))
    g = torch.Generator(device=dev).manual_seed(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ews = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)     # zeroed workspace (rx.h header)

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(a.iters):
            flush.fill_(1)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        return ts[len(ts) // 2]

    if a.kind == "decode" and a.cascade:
        # C5-style step: B requests share `cascade` cached tokens, each owns seq - cascade more
        L, P = a.seq, a.cascade
        S = P + B * (L - P) + 16
        kp = torch.randn((S, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vp = torch.randn_like(kp)
        rtt = torch.zeros((B, L), dtype=torch.int32, device=dev)
        rtt[:, :P] = torch.arange(1, P + 1, dtype=torch.int32, device=dev)
        own = torch.arange(P + 1, P + 1 + B * (L - P), dtype=torch.int32, device=dev).view(B, L - P)
        rtt[:, P:] = own
        new = own[:, -1].contiguous()
        q = torch.randn((B, h_q, hd), device=dev, generator=g).to(torch.bfloat16)
        kn = torch.randn((B, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vn = torch.randn_like(kn)
        o = torch.empty_like(q)
        lens = torch.full((B,), L, dtype=torch.int32, device=dev)
        ws = torch.zeros(max(rx.rx_decode_cascade_workspace_bytes(cfg, B, L, P),
                             rx.rx_decode_workspace_bytes(cfg, B, L)) + 1, dtype=torch.uint8, device=dev)
        ms_c = timeit(lambda: rx.rx_decode_cascade_append(cfg, rtt, None, lens, L, P, q, kn, vn, new, kp, vp, o, ws))
        ms_p = timeit(lambda: rx.rx_decode_append(cfg, rtt, None, lens, L, q, kn, vn, new, kp, vp, o, ws))
        uniq = (P + B * (L - P)) * h_kv * hd * 4
        flops = 4 * hd * h_q * B * L
        print(f"decode-step {h_q}/{h_kv}/{hd} B={B} L={L} shared={P}: cascade {ms_c*1e3:.1f} us "
              f"({uniq/ms_c/1e6:.0f} GB/s unique, {flops/ms_c/1e9:.1f} TFLOP/s)  vs per-request {ms_p*1e3:.1f} us "
              f"-> {ms_p/ms_c:.2f}x")
    elif a.kind == "decode":
        L = a.seq
        S = (L if a.shared_prefix else B * L) + 16
        kp = torch.randn((S, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vp = torch.randn_like(kp)
        if a.shared_prefix:
            rtt = torch.arange(1, L + 1, dtype=torch.int32, device=dev).repeat(B, 1)
        else:
            base = torch.arange(B * L, dtype=torch.int32, device=dev) + 1
            if a.scatter:
                base = base[torch.randperm(B * L, device=dev, generator=g)]
            rtt = base.view(B, L).contiguous()
        q = torch.randn((B, h_q, hd), device=dev, generator=g).to(torch.bfloat16)
        o = torch.empty_like(q)
        lens = torch.full((B,), L, dtype=torch.int32, device=dev)
        ws = torch.zeros(rx.rx_decode_workspace_bytes(cfg, B, L) + 1, dtype=torch.uint8, device=dev)
        ms = timeit(lambda: rx.rx_decode(cfg, rtt, None, lens, L, q, kp, vp, o, ws))
        uniq = (L if a.shared_prefix else B * L)
        byt = uniq * h_kv * hd * 4 + 2 * B * h_q * hd * 2 + 4 * B * L
        logical = B * L * h_kv * hd * 4
        print(f"decode {h_q}/{h_kv}/{hd} B={B} L={L}: {ms*1e3:.1f} us  alg {byt/ms/1e6:.0f} GB/s  "
              f"logical {logical/ms/1e6:.0f} GB/s  tokens/s {B/ms*1e3:.3e}")
    elif a.kind == "extend" and (a.ragged or a.half):
        import numpy as np
        r = np.random.default_rng(0)
        Ps = r.integers(a.prefix // 2, a.prefix * 3 // 2 + 1, B) if a.ragged else np.full(B, a.prefix)
        Es = r.integers(a.ext * 2 // 3, a.ext * 4 // 3 + 1, B) if a.ragged else np.full(B, a.ext)
        tot = int((Ps + Es).sum())
        S = tot + 16
        kp = torch.randn((S, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vp = torch.randn_like(kp)
        stride = int((Ps + Es).max())
        rtt_h = np.zeros((B, stride), dtype=np.int32)
        base = 1
        for b in range(B):
            n = int(Ps[b] + Es[b])
            rtt_h[b, :n] = np.arange(base, base + n)
            base += n
        if a.half:       # every other 384-token run of every prefix: slots permuted across requests
            mask = np.zeros((B, stride), dtype=bool)
            for b in range(B):
                for s0 in range(384, int(Ps[b]), 768):
                    mask[b, s0:min(s0 + 384, int(Ps[b]))] = True
            vals = rtt_h[mask]
            rtt_h[mask] = vals[r.permutation(len(vals))]
        rtt = torch.from_numpy(rtt_h).to(dev)
        N = int(Es.sum())
        q = torch.randn((N, h_q, hd), device=dev, generator=g).to(torch.bfloat16)
        kn = torch.randn((N, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vn = torch.randn_like(kn)
        o = torch.empty_like(q)
        pre = torch.from_numpy(Ps.astype(np.int32)).to(dev)
        ext = torch.from_numpy(Es.astype(np.int32)).to(dev)
        ind = torch.from_numpy(np.concatenate([[0], np.cumsum(Es)]).astype(np.int32)).to(dev)
        ms = timeit(lambda: rx.rx_extend(cfg, rtt, None, pre, ext, ind, N, int(Es.max()), int(Ps.max()), q, kn, vn,
                                         kp, vp, o, ews))
        flops = 4 * hd * h_q * float(np.sum(Es * Ps + Es * (Es + 1) / 2))
        print(f"extend {h_q}/{h_kv}/{hd} B={B} P~{a.prefix} E~{a.ext} ragged={a.ragged} half={a.half}: "
              f"{ms*1e3:.1f} us  {flops/ms/1e9:.1f} TFLOP/s tokens/s {N/ms*1e3:.3e}")
    elif a.kind == "extend":
        P, E = a.prefix, a.ext
        S = P + B * E + 16 if a.shared_prefix else B * (P + E) + 16
        kp = torch.randn((S, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vp = torch.randn_like(kp)
        rtt = torch.zeros((B, P + E), dtype=torch.int32, device=dev)
        for b in range(B):
            if a.shared_prefix:
                rtt[b, :P] = torch.arange(1, P + 1)
                rtt[b, P:] = torch.arange(P + 1 + b * E, P + 1 + (b + 1) * E)
            else:
                rtt[b] = torch.arange(1 + b * (P + E), 1 + (b + 1) * (P + E))
        if a.scatter:   # fragmented prefix slots (every tile takes the tile::gather4 path)
            pre = rtt[:, :P].reshape(-1)
            rtt[:, :P] = pre[torch.randperm(pre.numel(), device=dev, generator=g)].view(B, P)
        N = B * E
        q = torch.randn((N, h_q, hd), device=dev, generator=g).to(torch.bfloat16)
        kn = torch.randn((N, h_kv, hd), device=dev, generator=g).to(torch.bfloat16)
        vn = torch.randn_like(kn)
        o = torch.empty_like(q)
        pre = torch.full((B,), P, dtype=torch.int32, device=dev)
        ext = torch.full((B,), E, dtype=torch.int32, device=dev)
        ind = torch.arange(B + 1, dtype=torch.int32, device=dev) * E
        ms = timeit(lambda: rx.rx_extend(cfg, rtt, None, pre, ext, ind, N, E, P, q, kn, vn, kp, vp, o, ews))
        flops = 4 * hd * h_q * B * (E * P + E * (E + 1) / 2)
        print(f"extend {h_q}/{h_kv}/{hd} B={B} P={P} E={E}: {ms*1e3:.1f} us  {flops/ms/1e9:.1f} TFLOP/s "
              f"tokens/s {N/ms*1e3:.3e}")


if __name__ == "__main__":
    main()
