"""dev probe: timeline of the extend-input H2D copies in an e2e C3 pass (start / duration relative
to the pass start) and of the extend kernels' waits."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import make_workload
from paper_2312_07104_b200.engine import Engine, plan_and_bank
from paper_2312_07104_b200 import hostio
from paper_2312_07104_b200.hostio import HostInputs

wl = make_workload("C3")
dev = torch.device("cuda", 0)
plan, bank = plan_and_bank(wl, dev)
eng = Engine(wl, dev)
hb = HostInputs(bank, dev)
marks = []
orig = hostio._Prefetcher._issue
def issue(self, i):
    fresh = i < len(self.lst) and i not in self.pending
    if fresh:
        a = torch.cuda.Event(True); a.record(self.stream)
    orig(self, i)
    if fresh:
        b = torch.cuda.Event(True); b.record(self.stream)
        marks.append((i, a, b))
hostio._Prefetcher._issue = issue
gets = []
orig_get = hostio._Prefetcher.__getitem__
def get(self, i):
    import time
    th = time.perf_counter()
    r = orig_get(self, i)
    e = torch.cuda.Event(True); e.record()
    gets.append((i, e, th))
    return r
hostio._Prefetcher.__getitem__ = get
import paper_2312_07104_b200.engine as E
orig_pinned = E.Engine._pinned
def pinned(self, name, n):
    import time
    t = time.perf_counter()
    r = orig_pinned(self, name, n)
    dt = time.perf_counter() - t
    if dt > 1e-3:
        print(f"    host: _pinned({name}, {n}) took {dt*1e3:.1f} ms")
    return r
E.Engine._pinned = pinned
ext_only = types.SimpleNamespace(ext=hb.ext, dec=bank.dec)
import time
for it in range(3):
    marks.clear(); gets.clear()
    th0 = time.perf_counter()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(True); t0.record()
    hb.reset(); eng.reset(); eng.enable_timing(True); eng.timer = []
    eng.run_workload(ext_only)
    t1 = torch.cuda.Event(True); t1.record()
    torch.cuda.synchronize()
    print(f"pass {t0.elapsed_time(t1):.1f} ms")
    for i, a, b in marks:
        print(f"  ext {i}: copy start {t0.elapsed_time(a):7.1f} ms  dur {a.elapsed_time(b):6.1f} ms  ({sum(t.numel()*t.element_size() for t in hb.ext.lst[i])/1e9:.2f} GB)")
    for i, e, th in gets:
        print(f"  compute stream past get({i}) at {t0.elapsed_time(e):7.1f} ms (host called it at {1e3*(th-th0):7.1f} ms)")
    for kind, a, b, *_ in eng.timer:
        if kind == "extend":
            print(f"  extend kernel at {t0.elapsed_time(a):7.1f} ms, {a.elapsed_time(b):6.2f} ms")
