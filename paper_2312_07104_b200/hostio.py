"""Host-resident inputs and outputs for the engine, overlapped with the kernels.

A serving process receives each attention call's q / k_new / v_new from the host and returns its
output to the host.  ``HostInputs`` keeps every call's inputs in pinned host memory and copies
them host->device on a dedicated copy stream ``depth`` calls ahead of use (the compute stream waits
on a per-call event); ``HostSink`` copies every output device->host on a second stream as soon as
the call that produced it retires.  Both directions of PCIe run concurrently with the kernels, so
an end-to-end step costs max(kernels, H2D, D2H) instead of their sum.  Plumbing only: no method
arithmetic.
"""
from __future__ import annotations

import torch


class _Prefetcher:
    """Indexable like a list of (q, k, v) device tensors; element i is copied ahead of use."""

    def __init__(self, host_list, device, depth, stream):
        self.lst = host_list
        self.dev = device
        self.depth = depth
        self.stream = stream
        self.pending = {}
        self.h2d_bytes = sum(t.numel() * t.element_size() for tr in host_list for t in tr)

    def reset(self):
        self.pending.clear()

    def _issue(self, i):
        if i >= len(self.lst) or i in self.pending:
            return
        with torch.cuda.stream(self.stream):
            ts = tuple(t.to(self.dev, non_blocking=True) for t in self.lst[i])
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending[i] = (ts, ev)

    def __getitem__(self, i):
        for j in range(i, i + self.depth):
            self._issue(j)
        ts, ev = self.pending.pop(i)
        cur = torch.cuda.current_stream()
        cur.wait_event(ev)
        for t in ts:
            t.record_stream(cur)           # the allocator must not recycle them before `cur` is done
        return ts


class HostInputs:
    """Drop-in for ``engine.InputBank`` with the tensors in pinned host memory."""

    def __init__(self, bank, device, ext_depth=2, dec_depth=16):
        self.stream = torch.cuda.Stream(device=device)
        hext = [tuple(t.cpu().pin_memory() for t in tr) for tr in bank.ext]
        hdec = [tuple(t.cpu().pin_memory() for t in tr) for tr in bank.dec]
        self.ext = _Prefetcher(hext, device, ext_depth, self.stream)
        self.dec = _Prefetcher(hdec, device, dec_depth, self.stream)

    @property
    def h2d_bytes(self):
        return self.ext.h2d_bytes + self.dec.h2d_bytes

    def reset(self):
        self.ext.reset()
        self.dec.reset()
        # nothing is copied before the caller's current stream reaches this point (timed regions)
        self.stream.wait_stream(torch.cuda.current_stream())


class HostSink:
    """Engine ``sink``: output of call i -> out_host[i] (pinned), D2H on its own stream."""

    def __init__(self, out_host, device):
        self.out = out_host
        self.stream = torch.cuda.Stream(device=device)
        self.i = 0
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in out_host)

    def reset(self):
        self.i = 0

    def __call__(self, kind, o):
        dst = self.out[self.i]
        self.i += 1
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            if o.is_contiguous():
                dst.view(o.shape).copy_(o, non_blocking=True)
            else:                              # TP all-gather result is a strided view
                dst.copy_(o.reshape(dst.shape), non_blocking=True)
        o.record_stream(self.stream)

    def join(self):
        """Make the current stream wait for every queued D2H copy (end of a timed region)."""
        torch.cuda.current_stream().wait_stream(self.stream)
