"""Where does the end-to-end (host I/O) C3 step lose time? (dev tool)  Times one workload pass with
inputs resident / prefetched from pinned host memory, with and without the D2H output sink."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from bench import make_workload
from paper_2312_07104_b200.engine import Engine, plan_and_bank
from paper_2312_07104_b200.hostio import HostInputs, HostSink


def main():
    wl = make_workload(sys.argv[1] if len(sys.argv) > 1 else "C3")
    dev = torch.device("cuda", 0)
    plan, bank = plan_and_bank(wl, dev)
    eng = Engine(wl, dev)
    hb = HostInputs(bank, dev)
    sink = HostSink([torch.empty((len(c.hashes), wl.shape.h_q, wl.shape.head_dim), dtype=torch.bfloat16,
                                 pin_memory=True) for c in plan.calls], dev)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)
    # "copy||": every H2D block copy issued up front on the copy streams while the kernels run from
    # the device-resident bank (no dependency): do copies and kernels overlap at all?
    def all_copies():
        for i in range(len(hb.ext.lst)):
            hb.ext._issue(i)
        for j in range(len(hb.dec.ranges)):
            hb.dec._issue(j)
    import types
    ext_only = types.SimpleNamespace(ext=hb.ext, dec=bank.dec)      # extend inputs via H2D only
    dec_only = types.SimpleNamespace(ext=bank.ext, dec=hb.dec)      # decode inputs via H2D only
    for name, inputs, sk in (("device", bank, None), ("copy||", bank, None), ("h2d", hb, None),
                             ("h2d-ext", ext_only, None), ("h2d-dec", dec_only, None),
                             ("d2h", bank, sink), ("both", hb, sink)):
        eng.sink = sk
        ts = []
        for i in range(4):
            flush.fill_(1)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            sink.reset()
            a.record()
            if inputs is not bank:
                hb.reset()
            if name == "copy||":
                all_copies()
            eng.reset()
            eng.run_workload(inputs)
            if sk is not None:
                sk.join()
            if name == "copy||":
                for st in hb.streams:
                    torch.cuda.current_stream().wait_stream(st)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"{name:7s}: {' '.join(f'{t:7.1f}' for t in ts)} ms")


if __name__ == "__main__":
    main()
