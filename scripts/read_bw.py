"""Read-only HBM bandwidth of this B200 (dev tool): torch reductions over a 4 GB buffer (a
read-only stream; MEASURED_PEAKS.json's hbm_gbs is a copy = read + write), and decode-kernel
probes: the same bytes as 8 kv heads x 256 requests vs 1 kv head x 2048 requests (each CTA's rows
contiguous), to see whether the [slot, head, dim] pool layout costs DRAM efficiency."""
import math
import os
import subprocess
import sys

import torch


def main():
    dev = torch.device("cuda", 0)
    x = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    x.fill_(1)
    xf = x.view(torch.float32)
    for name, fn in (("sum fp32", lambda: xf.sum()), ("amax fp32", lambda: xf.amax())):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ts.sort()
        print(f"{name}: {x.numel() / (ts[5] / 1e3) / 1e9:.0f} GB/s read")
    del x, xf
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for h in (["32", "8", "128", "--batch", "256"], ["4", "1", "128", "--batch", "2048"],
              ["32", "8", "128", "--batch", "256", "--scatter"]):
        out = subprocess.run([sys.executable, os.path.join(root, "scripts", "kbench.py"), "decode", "--h", *h,
                              "--seq", "2048"], capture_output=True, text=True).stdout.strip().splitlines()
        print(out[-1] if out else "(no output)")


if __name__ == "__main__":
    main()
