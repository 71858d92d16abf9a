"""Host-resident inputs and outputs for the engine, overlapped with the kernels.

A serving process receives each attention call's q / k_new / v_new from the host and returns its
output to the host.  ``HostInputs`` keeps every call's inputs in pinned host memory and copies
them host->device on dedicated copy streams ``depth`` calls ahead of use (the compute stream waits
on a per-call event); ``HostSink`` copies every output device->host on a second stream as soon as
the call that produced it retires.  Both directions of PCIe run concurrently with the kernels, so
an end-to-end step costs max(kernels, H2D, D2H) instead of their sum.  Plumbing only: no method
arithmetic.
"""
from __future__ import annotations

import torch


def _aligned(nb):
    return (nb + 255) // 256 * 256


class _Prefetcher:
    """Indexable like a list of (q, k, v) device tensors; element i is copied ahead of use into a
    preallocated device ring of depth + 1 slots (no allocation per call: a caching-allocator miss
    on a ~1 GB extend input can stall the host behind the device).  Slot reuse waits on an event
    recorded on the compute stream once the previous call that used the slot was enqueued."""

    def __init__(self, host_list, device, depth, stream):
        self.lst = host_list
        self.dev = device
        self.depth = depth
        self.stream = stream
        self.pending = {}
        self.h2d_bytes = sum(t.numel() * t.element_size() for tr in host_list for t in tr)
        cap = max([sum(_aligned(t.numel() * t.element_size()) for t in tr) for tr in host_list] or [256])
        self.nslots = depth + 1
        self.ring = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(self.nslots)]
        self.free = [None] * self.nslots

    def reset(self):
        self.pending.clear()

    def _issue(self, i):
        if i >= len(self.lst) or i in self.pending:
            return
        slot = i % self.nslots
        buf = self.ring[slot]
        with torch.cuda.stream(self.stream):
            if self.free[slot] is not None:
                self.stream.wait_event(self.free[slot])
            views, off = [], 0
            for t in self.lst[i]:
                nb = t.numel() * t.element_size()
                v = buf[off:off + nb].view(t.dtype).view(t.shape)
                v.copy_(t, non_blocking=True)
                views.append(v)
                off += _aligned(nb)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending[i] = (tuple(views), ev)

    def __getitem__(self, i):
        cur = torch.cuda.current_stream()
        if i > 0:
            # call i - 1 is fully enqueued: its slot is free once the compute stream gets here
            ev = torch.cuda.Event()
            ev.record(cur)
            self.free[(i - 1) % self.nslots] = ev
        for j in range(i, i + self.depth):
            self._issue(j)
        ts, ev = self.pending.pop(i)
        cur.wait_event(ev)
        return ts


class _BlockPrefetcher:
    """Like _Prefetcher for many small calls (decode steps): the calls' tensors live back to back in
    ONE pinned byte buffer and are copied `block` calls per cudaMemcpy, `depth` blocks ahead, into a
    device ring of depth + 1 block buffers, so the host issues one copy per block instead of three
    per call and nothing is allocated per block."""

    def __init__(self, host_list, device, block, depth, stream):
        self.dev, self.block, self.depth, self.stream = device, block, depth, stream
        self.meta = []                         # per call: [(byte offset, nbytes, dtype, shape)]
        off = 0
        for tr in host_list:
            m = []
            for t in tr:
                nb = t.numel() * t.element_size()
                m.append((off, nb, t.dtype, tuple(t.shape)))
                off += _aligned(nb)
            self.meta.append(m)
        self.h2d_bytes = sum(t.numel() * t.element_size() for tr in host_list for t in tr)
        self.buf = torch.empty(max(off, 1), dtype=torch.uint8, pin_memory=True)
        for tr, m in zip(host_list, self.meta):
            for t, (o, nb, _, _) in zip(tr, m):
                self.buf[o:o + nb].copy_(t.reshape(-1).view(torch.uint8))
        n = len(host_list)
        self.ranges = []                       # per block: (first byte, end byte)
        for b0 in range(0, n, block):
            b1 = min(n, b0 + block)
            first = self.meta[b0][0][0]
            last = self.meta[b1 - 1][-1]
            self.ranges.append((first, last[0] + last[1]))
        cap = max([b - a for a, b in self.ranges] or [256])
        self.nslots = depth + 1
        self.ring = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(self.nslots)]
        self.free = [None] * self.nslots
        self.pending = {}

    def reset(self):
        self.pending.clear()

    def _issue(self, j):
        if j >= len(self.ranges) or j in self.pending:
            return
        a, b = self.ranges[j]
        slot = j % self.nslots
        with torch.cuda.stream(self.stream):
            if self.free[slot] is not None:
                self.stream.wait_event(self.free[slot])
            d = self.ring[slot][:b - a]
            d.copy_(self.buf[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        self.pending[j] = (d, ev, a, False)

    def __getitem__(self, i):
        j = i // self.block
        cur = torch.cuda.current_stream()
        if i % self.block == 0 and j > 0:
            # every call of block j - 1 is enqueued: its slot is free once the compute stream gets here
            ev = torch.cuda.Event()
            ev.record(cur)
            self.free[(j - 1) % self.nslots] = ev
        for k in range(j, j + self.depth):
            self._issue(k)
        d, ev, a, waited = self.pending[j]
        if not waited:
            cur.wait_event(ev)
            self.pending[j] = (d, ev, a, True)
        out = tuple(d[o - a:o - a + nb].view(dt).view(shape) for o, nb, dt, shape in self.meta[i])
        if i % self.block == self.block - 1 or i == len(self.meta) - 1:
            self.pending.pop(j)
        return out


class HostInputs:
    """Drop-in for ``engine.InputBank`` with the tensors in pinned host memory."""

    def __init__(self, bank, device, ext_depth=None, dec_block=None, dec_depth=None):
        # ext_depth 1: the next turn's extend input is queued on the copy engines only when the
        # host reaches that turn, i.e. AFTER the current turn's decode-input blocks (the engines
        # serve copies in submission order); 2 (the next extend at once) measured 506 vs 483 ms
        # per C3 pass with host I/O.  RX_EXT_DEPTH / RX_DEC_BLOCK / RX_DEC_DEPTH: A/B knobs.
        import os
        ext_depth = ext_depth if ext_depth is not None else int(os.environ.get("RX_EXT_DEPTH", "1"))
        dec_block = dec_block if dec_block is not None else int(os.environ.get("RX_DEC_BLOCK", "16"))
        dec_depth = dec_depth if dec_depth is not None else int(os.environ.get("RX_DEC_DEPTH", "8"))
        # one copy stream per call kind: a large extend prefetch (~1 GB for a C3 turn) must not
        # queue in front of the small per-step decode inputs that are needed first
        self.streams = (torch.cuda.Stream(device=device), torch.cuda.Stream(device=device))
        hext = [tuple(t.cpu().pin_memory() for t in tr) for tr in bank.ext]
        hdec = [tuple(t.cpu().pin_memory() for t in tr) for tr in bank.dec]
        self.ext = _Prefetcher(hext, device, ext_depth, self.streams[0])
        self.dec = _BlockPrefetcher(hdec, device, dec_block, dec_depth, self.streams[1])

    @property
    def h2d_bytes(self):
        return self.ext.h2d_bytes + self.dec.h2d_bytes

    def reset(self):
        self.ext.reset()
        self.dec.reset()
        # nothing is copied before the caller's current stream reaches this point (timed regions)
        for st in self.streams:
            st.wait_stream(torch.cuda.current_stream())


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
