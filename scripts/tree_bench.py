"""Host radix-tree cost (the P:437 analog: "the time used for managing the RadixAttention data
structures is only 0.2 seconds" of 74.3 s): one plan pass of a workload — every match_prefix,
inc_ref, alloc/evict, dec_ref, insert (and rx_schedule waves) with no kernels — through the C++
library and through the Python oracle tree, on the host cores.  CPU only.

    python scripts/tree_bench.py [C3|C4|C5|MIX|JSON] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import make_workload
from oracle.driver import OracleEngine
from paper_2312_07104_b200.engine import Engine
from rxgen import workloads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C3")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    extra = {"C4": workloads.c4, "MIX": workloads.mix, "JSON": workloads.json_decode}
    wl = extra[a.workload]() if a.workload in extra else make_workload(a.workload)
    rec = Engine(wl, plan_only=True, record=True)
    rec.run_workload()
    ops = sum(1 for t in rec.trace if t[0] in ("match", "inc_ref", "alloc", "evict", "dec_ref", "insert"))
    best_lib, best_lib_tree = 1e9, 1e9
    e = Engine(wl, plan_only=True)
    e.collect_calls = False                # tree ops only: no per-call input bookkeeping
    e.run_workload()                       # first pass also draws the mock-model token streams (cached)
    for _ in range(a.reps):
        e.reset()
        e.calls = []
        t0 = time.perf_counter()
        e.run_workload()
        best_lib = min(best_lib, time.perf_counter() - t0)
        best_lib_tree = min(best_lib_tree, e.stats["tree_s"])
    o = OracleEngine(wl)
    t0 = time.perf_counter()
    o.run_workload()                       # (includes the oracle's own token-stream generation)
    t_or = time.perf_counter() - t0
    print(json.dumps({"workload": wl.name, "tree_ops": ops,
                      "library_pass_s": best_lib, "library_tree_s": best_lib_tree,
                      "library_tree_ops_per_s": ops / best_lib_tree,
                      "oracle_pass_s": t_or, "oracle_tree_ops_per_s": ops / t_or,
                      "note": "library_tree_s = engine time in tree sections (C calls + their numpy marshalling);"
                              " pass = the whole plan pass incl. request bookkeeping"}))


if __name__ == "__main__":
    main()
