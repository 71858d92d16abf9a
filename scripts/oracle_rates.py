"""Oracle throughput per config (BASELINE.md §6 "Oracle tokens/s"): the CPU oracle (oracle/, fp64,
Python radix tree) as it stands over the WHOLE workload's tree flow, with sampled attention rows
(every `ext_every`-th extend row, every `dec_every`-th decode step plus the last) whose time is
extrapolated to every row.  Input generation is timed and excluded (the GPU arm's inputs are
pre-generated).  One process (cores = 1); a dev tool, run on the bench box's host.

    python scripts/oracle_rates.py [C1 C2 C4 C5] [--ext-every 64] [--dec-every 16]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.driver import OracleEngine  # noqa: E402
from rxgen import workloads  # noqa: E402


def rate(name, ext_every, dec_every):
    import torch
    from threadpoolctl import threadpool_limits
    torch.set_num_threads(1)
    threadpool_limits(1)
    wl = workloads.CONFIGS[name]()

    class Timed(OracleEngine):
        def _store(self, slots, hashes):
            t = time.perf_counter()
            super()._store(slots, hashes)
            self.t_input += time.perf_counter() - t

        def _q(self, h, heads):
            t = time.perf_counter()
            r = super()._q(h, heads)
            self.t_input += time.perf_counter() - t
            return r

        def _attend(self, seq, p):
            t, t_in = time.perf_counter(), self.t_input
            r = super()._attend(seq, p)
            self.t_att[self.phase] += time.perf_counter() - t - (self.t_input - t_in)   # q generation excluded
            return r

    cnt = {"ext": 0, "ext_s": 0, "dec": 0, "dec_s": 0}

    def se(call, seqs):
        oe.phase = "ext"
        rows = [(i, j) for i, q in enumerate(seqs) for j in range(q.n_prompt - q.prefix_len)]
        pick = rows[::ext_every]
        cnt["ext"] += len(rows)
        cnt["ext_s"] += len(pick)
        return pick

    def sd(call, step, running):
        oe.phase = "dec"
        cnt["dec"] += len(running)
        last = all(len(q.tokens) - q.n_prompt >= q.n_out for q in running)
        if step % dec_every == 0 or last:
            cnt["dec_s"] += len(running)
            return list(range(len(running)))
        return []

    materialize = wl.num_slots * wl.shape.h_kv * wl.shape.head_dim <= (1 << 28)
    oe = Timed(wl, se, sd, materialize=materialize)
    oe.t_input, oe.t_att, oe.phase = 0.0, {"ext": 0.0, "dec": 0.0}, "ext"
    t0 = time.perf_counter()
    oe.run_workload()
    wall = time.perf_counter() - t0
    other = wall - oe.t_input - oe.t_att["ext"] - oe.t_att["dec"]
    t_ext = oe.t_att["ext"] * cnt["ext"] / max(1, cnt["ext_s"])
    t_dec = oe.t_att["dec"] * cnt["dec"] / max(1, cnt["dec_s"])
    est = other + t_ext + t_dec
    return {"config": name, "tokens": cnt["ext"] + cnt["dec"], "tokens_per_s": (cnt["ext"] + cnt["dec"]) / est,
            "extend_tokens_per_s": cnt["ext"] / max(1e-9, t_ext + other * cnt["ext"] / max(1, cnt["ext"] + cnt["dec"])),
            "decode_tokens_per_s": cnt["dec"] / max(1e-9, t_dec + other * cnt["dec"] / max(1, cnt["ext"] + cnt["dec"])),
            "cores": 1, "extrapolated": True, "sampled_rows": cnt["ext_s"] + cnt["dec_s"],
            "wall_s": wall, "tree_and_bookkeeping_s": other}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C4", "C5"])
    ap.add_argument("--ext-every", type=int, default=64)
    ap.add_argument("--dec-every", type=int, default=16)
    a = ap.parse_args()
    for c in a.configs:
        ee = 1 if c == "C1" else a.ext_every
        de = 1 if c == "C1" else a.dec_every
        print(json.dumps(rate(c, ee, de)), flush=True)


if __name__ == "__main__":
    main()
