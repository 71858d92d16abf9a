"""bench.py — attention tokens/s of the RadixAttention hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (TP over KV heads, NCCL all-gather)

One STEP = one pass of the whole hot path over the
workload: every radix-tree op (match_prefix, inc_ref, alloc/evict, dec_ref,
insert — host C++ via the C ABI), every req_to_token upload, every KV store,
extend and decode launch (and at N > 1 the per-call all-gather).  Inputs
(q / k_new / v_new of every call) are generated from the workload BEFORE
timing and are resident in HBM.  L2 is flushed (a write of 2x the L2 size)
before every timed step; each step is bracketed by barrier + synchronize and
timed with CUDA events on the launching stream; the max over ranks is taken.

value = (extend tokens + decode tokens) of the whole job / time  [tokens/s]
e2e   = the same with q/k/v copied host->device (pinned) per call and every
        output copied device->host inside the timed region.

configs: C1, C2, C4, C5 under the same protocol (min(K, 5) steps, 3 warm-up),
per phase: extend tokens/s and TFLOP/s against the bf16 peak; decode tokens/s
and GB/s on unique (a shared prefix once) and logical bytes against HBM.

--impl reference: the CPU oracle (oracle/, fp64, Python tree) on the host
cores (this tier's reference arm): a process pool with one worker per core,
each running one whole C3 session of the same workload (sessions share
nothing, so a session is an exact share of the run) with sampled attention
rows extrapolated to every row (labelled).  cpu_baseline is one such pool
step with denser sampling.  Only these two legs execute oracle/ code.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def make_workload(name, scale=None):
    from rxgen import workloads
    if name == "C3":
        return workloads.c3()
    if name == "C5":
        return workloads.c5()
    if name == "C2":
        return workloads.c2()
    if name == "C1":
        return workloads.c1()
    if name == "C4":
        return workloads.c4()
    raise ValueError(name)


# ------------------------------------------------------------------ CPU oracle (reference arm / cpu_baseline)
METRIC = "attn tokens/s (extend+decode), one attention layer"     # both arms (BASELINE.json metric)


def _session_workload(full, s, num_slots=8192):
    """Session s of the C3 workload as a workload of its own: C3 sessions share nothing (SURVEY
    §8(d)), so a session's tree ops, stores and attention rows are exactly its share of the full
    run (same prompts, same prefix hashes, hence the same K/V/Q values); only slot numbers differ."""
    from rxgen.workloads import Workload
    m = dict(full.meta)
    m["turn_inputs"] = [full.meta["turn_inputs"][s]]
    m["turn_outputs"] = [full.meta["turn_outputs"][s]]
    return Workload(full.name, full.shape, num_slots, full.vocab, full.seed, [], m)


def _oracle_session(args):
    """Worker: the oracle (as it stands) over one C3 session, every extend row `ext_every`-th and
    every `dec_every`-th decode step (plus the last) attended; attention time extrapolated to every
    row.  Input generation (K/V values written into the oracle's pool, q values) is timed and
    excluded, as the GPU arm's inputs are pre-generated.  Returns (rows, extrapolated s, wall s)."""
    s, ext_every, dec_every = args
    import torch
    from threadpoolctl import threadpool_limits
    torch.set_num_threads(1)                  # one core per worker: BLAS and torch single-threaded
    threadpool_limits(1)
    from oracle.driver import OracleEngine
    from rxgen import workloads

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

    wl = _session_workload(workloads.c3(), s)
    oe = Timed(wl, se, sd, materialize=True)
    oe.t_input, oe.t_att, oe.phase = 0.0, {"ext": 0.0, "dec": 0.0}, "ext"
    t0 = time.perf_counter()
    oe.run_workload()
    wall = time.perf_counter() - t0
    other = wall - oe.t_input - oe.t_att["ext"] - oe.t_att["dec"]          # tree ops, bookkeeping
    est = (other + oe.t_att["ext"] * cnt["ext"] / max(1, cnt["ext_s"])
           + oe.t_att["dec"] * cnt["dec"] / max(1, cnt["dec_s"]))
    # sampled decode steps see the per-step work of the steps around them: the "last" rule adds
    # one step per turn, so the estimate is the sampled mean row cost x all rows
    return cnt["ext"] + cnt["dec"], est, wall, cnt


class OracleSampler:
    """The CPU oracle on the box's host cores: a process pool of one worker per core, each running
    one whole C3 session (all 4 turns, the full shapes) through the oracle's tree flow and
    attention, with sampled attention rows extrapolated to every row (labelled).  One `step` = one
    session per worker (sessions k*P .. k*P+P-1 of the 256); value = rows of those sessions / the
    slowest worker's extrapolated time (whole-pool throughput)."""

    def __init__(self, ext_every, dec_every, procs=None):
        import multiprocessing as mp
        self.P = procs or len(os.sched_getaffinity(0))
        self.ext_every, self.dec_every = ext_every, dec_every
        self.pool = mp.get_context("fork").Pool(self.P)
        self.k = 0

    def step(self):
        ss = [(self.k * self.P + i) % 256 for i in range(self.P)]
        self.k += 1
        t0 = time.perf_counter()
        res = self.pool.map(_oracle_session, [(s, self.ext_every, self.dec_every) for s in ss])
        wall = time.perf_counter() - t0
        rows = sum(r[0] for r in res)
        est = max(r[1] for r in res)
        sampled = sum(r[3]["ext_s"] + r[3]["dec_s"] for r in res)
        return rows, est, wall, sampled

    def close(self):
        self.pool.close()
        self.pool.join()

    def describe(self, rows, sampled, steps):
        return (f"oracle/ (fp64, Python radix tree) over {steps * self.P} whole C3 sessions (all 4 turns, full "
                f"shapes; {self.P} worker processes, one session each per step); {sampled} of {rows} attention "
                f"rows computed (every {self.ext_every}th extend row, every {self.dec_every}th decode step + the last "
                f"of each turn), attention time extrapolated to all rows; input generation excluded; tree ops "
                f"included")


def run_oracle_baseline(ext_every=4, dec_every=16):
    """cpu_baseline: one pool step, ~10-30 s."""
    smp = OracleSampler(ext_every, dec_every)
    try:
        rows, est, wall, sampled = smp.step()
    finally:
        smp.close()
    return {"value": rows / est, "unit": "tokens/s", "cores": smp.P, "kind": "oracle", "extrapolated": True,
            "sample": smp.describe(rows, sampled, 1) + f"; {wall:.1f} s wall"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]
        else:
            self.lines = []

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except Exception:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parallel", default="tp", choices=["tp", "dp"],
                    help="multi-GPU axis: tp = KV-head tensor parallelism (north star, default); dp = one "
                         "data-parallel replica per GPU behind the router meta-tree (App. A.4), few-shot workload")
    ap.add_argument("--configs", default="C1,C2,C4,C5",
                    help="also time these workloads under the same protocol (reported under 'configs'); 'none'")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        # this tier's reference arm: the CPU oracle, rank 0 only; one step = one
        # session per host core; C3 only (its sessions are independent, so a session is an exact
        # share of the workload)
        if rank != 0:
            return
        if args.workload != "C3":
            print(json.dumps({"impl": "reference", "unavailable": "the oracle arm samples C3 sessions only"}))
            return
        smp = OracleSampler(ext_every=16, dec_every=32)
        try:
            for _ in range(args.warmup):
                smp.step()
            rows = est = wall = sampled = 0
            for _ in range(args.steps):
                r, e, w, sm = smp.step()
                rows, est, wall, sampled = rows + r, est + e, wall + w, sampled + sm
        finally:
            smp.close()
        value = rows / est
        cpu = {"value": value, "unit": "tokens/s", "cores": smp.P, "kind": "oracle", "extrapolated": True,
               "sample": smp.describe(rows, sampled, args.steps)}
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1000.0 / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (rxgen, same C3 sessions as the GPU arm)",
                "config": {"workload": "C3", "shape_hq_hkv_hd": [32, 8, 128],
                           "sample": f"{smp.P} whole sessions per step, sampled rows, extrapolated"},
                "cpu_baseline": cpu,
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    if args.parallel == "dp":
        return run_dp(args, world, rank, local)

    import torch
    import torch.distributed as dist
    # RX_BENCH_TP_SELFTEST=1 under `torchrun --nproc-per-node 1`: run the TP code path (NCCL group,
    # per-call output all-gather, chunked extend gathers, max-over-ranks) on one GPU — a check of
    # the multi-GPU plumbing, not a scaling number
    tp_path = world > 1 or (os.environ.get("RX_BENCH_TP_SELFTEST") == "1" and "RANK" in os.environ)
    if tp_path:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    from paper_2312_07104_b200.tp import make_gather

    gather = make_gather() if tp_path else None
    peaks, peak_src = load_peaks()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)

    def barrier():
        if tp_path:
            dist.barrier()

    def max_over_ranks(ms):
        if not tp_path:
            return ms
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    with ClockSampler(torch.cuda.current_device()) as clk:
        main_run = measure(args.workload, args.steps, args.warmup, dev, rank, world, gather, flush, barrier,
                           max_over_ranks, peaks, keep=True)
    wl, plan, eng, bank = main_run.pop("_objs")
    kern = main_run["_kern"]
    total_ms = main_run["_total_ms"]
    tokens = main_run["tokens_per_step"]

    # dominant kernel by share of device time
    kind, (kms, knl, kcalls, kwork, _) = max(((k_, v_) for k_, v_ in kern.items() if k_ != "gather"),
                                             key=lambda kv: kv[1][0])
    per_launch_ms = kms / kcalls
    if kind == "extend":
        achieved = kwork / kcalls / (per_launch_ms / 1000.0) / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        roof = {"bound": "tensor", "unit": "TFLOP/s", "kernel": "rx_extend (extend_kernel)"}
    else:
        achieved = kwork / kcalls / (per_launch_ms / 1000.0) / 1e9
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "unit": "GB/s", "kernel": f"rx_{kind}"}
    # traffic: DRAM bytes per launch from the committed `ncu --set full` capture of this kernel in
    # this workload (profiles/r<k>_ncu_<kind>_traffic_<wl>.json, scripts/ncu_traffic.py), expressed for
    # this run's average launch: (captured DRAM bytes / captured algorithmic bytes) x algorithmic
    # bytes per launch here
    traffic, traffic_src = None, None
    tp = None
    for rnd in ("r2", "r1"):                          # the newest committed capture
        cand = os.path.join(ROOT, "profiles", f"{rnd}_ncu_{kind}_traffic_{wl.name}.json")
        if os.path.exists(cand):
            tp = cand
            break
    if tp is not None:
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj["traffic_over_algorithmic"] * (kwork / kcalls)
        traffic_src = {"file": os.path.relpath(tp, ROOT), "captured_launches": len(tj["launches"]),
                       "dram_bytes_per_captured_launch": tj["dram_bytes_per_launch"],
                       "algorithmic_bytes_per_captured_launch": tj["algorithmic_bytes_per_launch"],
                       "ratio": tj["traffic_over_algorithmic"],
                       "note": "per-rank shard at N > 1 (captured at N = 1)" if world > 1 else None}
    nominal = 2250.0 if kind == "extend" else 8000.0            # TFLOP/s dense bf16 | GB/s HBM3e
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": traffic,
                 "nominal_peak": nominal, "frac_nominal": achieved / nominal,
                 "traffic_source": traffic_src,
                 "peak_source": f"{peak_src} MEASURED_PEAKS.json" if peak_src == "measured" else "fallback",
                 "share_of_step": kms / total_ms})

    # ---------------------------------------------------------- e2e: host inputs, host outputs
    e2e = None
    if not args.no_e2e:
        from paper_2312_07104_b200.hostio import HostInputs, HostSink
        # every call's inputs live in pinned host memory and go host->device on a copy stream a few
        # calls ahead; every call's output lands in a preallocated pinned host buffer via a D2H
        # stream right after the call (paper_2312_07104_b200/hostio.py); sizes come from the plan.
        # At N > 1 every rank copies its own inputs in and rank 0 copies the gathered output out
        # (the other ranks' gathered copies are not needed on the host).
        hbank = HostInputs(bank, dev)
        h2d = hbank.h2d_bytes
        eng.enable_timing(False)
        hq = eng.hq * world
        sink = None
        if rank == 0:
            sink = HostSink([torch.empty((len(c.hashes), hq, wl.shape.head_dim), dtype=torch.bfloat16,
                                         pin_memory=True) for c in plan.calls], dev)
        d2h = sink.d2h_bytes if sink is not None else 0
        eng.sink = sink
        for _ in range(args.warmup):            # untimed, like the device-resident steps
            if sink is not None:
                sink.reset()
            hbank.reset()
            eng.reset()
            eng.run_workload(hbank)
            if sink is not None:
                sink.join()
        torch.cuda.synchronize()
        e2e_times = []
        for it in range(max(1, args.steps)):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            if sink is not None:
                sink.reset()
            a.record()
            hbank.reset()
            eng.reset()
            eng.run_workload(hbank)
            if sink is not None:
                sink.join()
            b.record()
            torch.cuda.synchronize()
            barrier()
            e2e_times.append(a.elapsed_time(b))
        eng.sink = None
        e_ms = max_over_ranks(sum(e2e_times))
        e2e = {"value": tokens * len(e2e_times) / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_ms / len(e2e_times),
               "note": "h2d counts every rank's inputs" if world > 1 else None}
        del hbank, sink
    del bank, eng, plan
    torch.cuda.empty_cache()

    # ---------------------------------------------------------- the other configs (same protocol)
    configs = {}
    if args.configs != "none":
        for name in [c for c in args.configs.split(",") if c and c != args.workload]:
            r = measure(name, min(args.steps, 5), max(3, min(args.warmup, 3)), dev, rank, world, gather, flush,
                        barrier, max_over_ranks, peaks, keep=False)
            for k_ in ("_objs", "_kern", "_total_ms"):
                r.pop(k_, None)
            configs[name] = r
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "C3":
        cpu = run_oracle_baseline()

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": main_run["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": main_run["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (rxgen: splitmix64 prefix-hash K/V/Q, mock-model tokens)",
            "config": {"workload": wl.name, "shape_hq_hkv_hd": [wl.shape.h_q, wl.shape.h_kv, wl.shape.head_dim],
                       "tokens_per_step": tokens, "extend_tokens": main_run["extend_tokens"],
                       "decode_tokens": main_run["decode_tokens"], "cache_hit_rate": main_run["cache_hit_rate"],
                       "parallelism": f"tp{world}" if world > 1 else ("tp1-selftest" if tp_path else "single"),
                       "l2_flush": "2x L2 write before each timed step", "num_slots": wl.num_slots},
            "gpu_launches": main_run["gpu_launches"], "roofline": roof, "kernels": main_run["kernels"],
            "tree_ms_per_step": main_run["tree_ms_per_step"],
            "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu, "configs": configs,
        }
        print(json.dumps(line))
    if tp_path:
        dist.destroy_process_group()


def run_dp(args, world, rank, local):
    """Data-parallel replicas (App. A.4): one worker per GPU, each with
    its own radix tree and pool, behind the router meta-tree.  Every rank replays the router and the
    other workers' tree operations on the host (plan-only shadows: deterministic, so every rank holds
    the same routing state with no communication) and runs its own worker's kernels; no data-path
    collective.  Workload rxgen.workloads.dp_fewshot: one hint per subject prefix (the router spreads
    them by load), then batches of interleaved few-shot questions the router sends to the worker that
    caches their subject.  Weak scaling (subjects and requests grow with the worker count).  One step
    = the whole workload from empty caches; value = tokens of ALL workers / max-over-ranks time."""
    import torch
    import torch.distributed as dist
    from paper_2312_07104_b200.dp import DPCluster
    from paper_2312_07104_b200.engine import InputBank
    from rxgen import workloads
    from rxgen.workloads import Request
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    base = workloads.dp_fewshot(workers=world)
    m = base.meta
    pres = {}
    for _, reqs in base.phases:
        for r in reqs:
            pres.setdefault(r.tag.split("s")[1].split("r")[0], r.prompt[:m["prefix"]])
    hints = [Request(pres[str(s_)].copy(), 0, f"hint{s_}") for s_ in range(m["subjects"])]
    wl = workloads.Workload("DP", base.shape, base.num_slots, base.vocab, base.seed,
                            [("dp_batch", hints)] + list(base.phases), m)
    lam = 0.1                   # affinity (1536 cached tokens) outweighs one batch's load imbalance
    plan = DPCluster(wl, world, plan_only=True, load_weight=lam)
    plan.run_workload()
    bank = InputBank(plan.workers[rank].calls, wl.shape, plan.workers[rank].heads_q, plan.workers[rank].heads_kv, dev)
    banks = [bank if w == rank else None for w in range(world)]
    cl = DPCluster(wl, world, device=dev, local=rank, load_weight=lam)
    flush = torch.empty(2 * torch.cuda.get_device_properties(dev).L2_cache_size, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        cl.reset()
        cl.run_workload(banks)
    torch.cuda.synchronize()
    times, launches = [], 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cl.reset()
            cl.run_workload(banks)
            b.record()
            torch.cuda.synchronize()
            barrier()
            times.append(a.elapsed_time(b))
            launches = cl.workers[rank].stats["launches"]
    ms = sum(times)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    st = [e.stats for e in plan.workers]
    tokens = sum(x["extend_tokens"] + x["decode_tokens"] for x in st)
    prompt = sum(x["prompt_tokens"] for x in st)
    cached = sum(x["cached_prompt_tokens"] for x in st)
    # W-worker optimum: each subject prefix computed once in the whole cluster (hint), every
    # question computed once, every later request hits its subject's prefix
    optimum_computed = m["subjects"] * m["prefix"] + sum(len(r.prompt) - m["prefix"] for _, rq in base.phases
                                                         for r in rq)
    per_worker = [int(x["prompt_tokens"]) for x in st]
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": tokens * len(times) / (ms / 1000.0), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (rxgen dp_fewshot: per-subject few-shot prefixes, mock-model tokens)",
            "config": {"workload": "DP few-shot (Llama-2-7B 32/32/128)", "parallelism": f"dp{world}",
                       "subjects": m["subjects"], "prefix": m["prefix"], "tokens_per_step": tokens,
                       "requests_per_step": sum(len(rq) for _, rq in wl.phases), "router_load_weight": lam,
                       "l2_flush": "2x L2 write before each timed step"},
            "cache_hit_rate": cached / prompt, "cache_hit_rate_optimal": 1.0 - optimum_computed / prompt,
            "prompt_tokens_per_worker": per_worker, "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": None, "note": "e2e / cpu_baseline / configs: see the default (tp) bench line"}))
    if world > 1:
        dist.destroy_process_group()


def measure(name, steps, warmup, dev, rank, world, gather, flush, barrier, max_over_ranks, peaks, keep):
    """One workload under the bench protocol: plan + inputs in HBM (untimed), `warmup` passes, then
    `steps` passes each bracketed by an L2 flush, barrier + synchronize and CUDA events on the
    launching stream; max over ranks.  Returns the per-config record (tokens/s overall and per
    phase, kernel figures against their rooflines)."""
    import torch
    from paper_2312_07104_b200.engine import Engine, plan_and_bank
    wl = make_workload(name)
    plan, bank = plan_and_bank(wl, dev, tp_rank=rank, tp_size=world)
    eng = Engine(wl, dev, tp_rank=rank, tp_size=world, gather=gather)
    tokens = plan.stats["extend_tokens"] + plan.stats["decode_tokens"]
    for _ in range(warmup):
        eng.reset()
        eng.run_workload(bank)
    torch.cuda.synchronize()
    times, kern, tree_s = [], {}, 0.0
    eng.enable_timing(True)
    for _ in range(steps):
        flush.fill_(1)
        barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        eng.timer = []
        a.record()
        eng.reset()
        eng.run_workload(bank)
        b.record()
        torch.cuda.synchronize()
        barrier()
        times.append(a.elapsed_time(b))
        tree_s += eng.stats["tree_s"]
        for k_, v_ in eng.timing_summary().items():
            t = kern.setdefault(k_, [0.0, 0, 0, 0.0, 0.0])
            for i in range(5):
                t[i] += v_[i]
    total_ms = max_over_ranks(sum(times))
    hbm, tf_peak = peaks["hbm_gbs"], peaks.get("bf16_tflops", 1662.5)
    phase_tokens = {"extend": plan.stats["extend_tokens"], "decode": plan.stats["decode_tokens"]}
    kernels = {}
    for k_, (ms, nl, calls, work, logical) in kern.items():
        sec = ms / 1000.0
        d = {"ms_per_step": ms / steps, "calls_per_step": calls // steps, "launches_per_step": nl // steps,
             "tokens_per_s": phase_tokens.get(k_, 0) * steps / sec if sec > 0 else None}
        if k_ == "gather":
            # TP output all-gather (kernel-only figures are the other entries): per gather call, and
            # per attention call (FusedGather: one barrier per decode run, the data moved by the
            # attention epilogue's own stores)
            att = sum(v_[2] for kk_, v_ in kern.items() if kk_ != "gather")
            d = {"ms_per_step": ms / steps, "calls_per_step": calls // steps,
                 "us_per_call": ms * 1000.0 / max(1, calls), "us_per_attention_call": ms * 1000.0 / max(1, att),
                 "kind": type(gather).__name__ if gather is not None else None}
            kernels[k_] = d
            continue
        if k_ == "extend":
            tf = work / sec / 1e12
            d.update({"tflops": tf, "frac_bf16_measured": tf / tf_peak, "frac_bf16_nominal": tf / 2250.0})
        else:
            gb, gl = work / sec / 1e9, logical / sec / 1e9
            d.update({"gbs": gb, "gbs_logical": gl, "frac_hbm_measured": gb / hbm, "frac_hbm_nominal": gb / 8000.0,
                      "note": "gbs: distinct pool rows once (a shared prefix counts once); gbs_logical: every "
                              "request's rows (paged-equivalent)"})
        kernels[k_] = d
    out = {"workload": wl.name, "shape_hq_hkv_hd": [wl.shape.h_q, wl.shape.h_kv, wl.shape.head_dim],
           "value": tokens * steps / (total_ms / 1000.0), "unit": "tokens/s", "ms_per_step": total_ms / steps,
           "steps": steps, "warmup": warmup, "tokens_per_step": tokens,
           "extend_tokens": plan.stats["extend_tokens"], "decode_tokens": plan.stats["decode_tokens"],
           "cache_hit_rate": plan.stats["cached_prompt_tokens"] / max(1, plan.stats["prompt_tokens"]),
           "kernels": kernels, "tree_ms_per_step": tree_s * 1000.0 / steps, "gpu_launches": eng.stats["launches"],
           "_kern": kern, "_total_ms": total_ms}
    if keep:
        out["_objs"] = (wl, plan, eng, bank)
    else:
        del eng, bank, plan
    return out


if __name__ == "__main__":
    main()
