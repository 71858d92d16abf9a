"""Pinned host<->device copy bandwidth on this box (dev tool): H2D alone, D2H alone, both at once on
separate streams, for 2 MB and 512 MB copies.  CUDA events; median of 5."""
import torch


def bw(fn, nbytes, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return nbytes / (ts[len(ts) // 2] / 1000) / 1e9


def main():
    dev = torch.device("cuda", 0)
    for size in (2 << 20, 512 << 20):
        n = 64 if size < (64 << 20) else 1
        h = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
        d = [torch.empty(size, dtype=torch.uint8, device=dev) for _ in range(n)]
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def h2d():
            for a, b in zip(d, h):
                a.copy_(b, non_blocking=True)

        def d2h():
            for a, b in zip(h, d):
                a.copy_(b, non_blocking=True)

        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                h2d_x()
            with torch.cuda.stream(s2):
                for a, b in zip(h2, d):
                    a.copy_(b, non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        h2 = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
        d2 = [torch.empty(size, dtype=torch.uint8, device=dev) for _ in range(n)]

        def h2d_x():
            for a, b in zip(d2, h):
                a.copy_(b, non_blocking=True)
        tot = size * n
        print(f"{size >> 20} MB x {n}: H2D {bw(h2d, tot):.1f} GB/s, D2H {bw(d2h, tot):.1f} GB/s, "
              f"both {bw(both, 2 * tot):.1f} GB/s (sum)")


if __name__ == "__main__" and __import__("sys").argv[-1] != "load":
    main()


def under_load():
    """H2D of 1 GiB pinned while another stream saturates HBM with reads (torch sum over 8 GiB):
    the rate the e2e path's input copies get while decode kernels run."""
    dev = torch.device("cuda", 0)
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    big = torch.ones(1 << 31, dtype=torch.float32, device=dev)
    s_load, s_copy = torch.cuda.Stream(), torch.cuda.Stream()
    for load in (False, True):
        torch.cuda.synchronize()
        if load:
            with torch.cuda.stream(s_load):
                for _ in range(40):
                    big.sum()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(s_copy):
            a.record()
            d.copy_(h, non_blocking=True)
            b.record()
        torch.cuda.synchronize()
        print(f"1 GiB H2D {'under HBM read load' if load else 'alone':20s}: {(1 << 30) / (a.elapsed_time(b) / 1000) / 1e9:.1f} GB/s")


if __name__ == "__main__" and __import__("sys").argv[-1] == "load":
    under_load()
