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

--impl reference: the CPU oracle (oracle/, fp64, Python tree) timed on a
bounded sample of the same workload on the host cores (this tier's reference
arm).  Only this leg and the cpu_baseline leg execute oracle/ code.
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
    raise ValueError(name)


# ------------------------------------------------------------------ CPU oracle (reference arm / cpu_baseline)
def oracle_sample(name):
    """Bounded sample of the workload for the CPU oracle (~10-30 s on the host cores)."""
    from rxgen import workloads
    if name == "C3":
        return workloads.c3(sessions=2, turns=2, num_slots=8192), "C3 shapes, 2 of 256 sessions x 2 of 4 turns, every row"
    if name == "C5":
        return workloads.c5(n_req=2, prefix=2048, decode=8, num_slots=8192), "C5 shapes, 2 of 128 requests, 2k of 8k context, 8 of 32 decode steps"
    if name == "C2":
        return workloads.c2(n_req=4, decode=8, num_slots=8192), "C2 shapes, 4 of 64 requests, 8 of 64 decode steps"
    return workloads.c1(), "C1 full"


def run_oracle(name):
    import torch
    from oracle.driver import OracleEngine
    torch.set_num_threads(len(os.sched_getaffinity(0)))
    wl, desc = oracle_sample(name)
    allr = lambda c, seqs: [(i, j) for i, s in enumerate(seqs) for j in range(s.n_prompt - s.prefix_len)]
    alld = lambda c, st, run: list(range(len(run)))
    t0 = time.perf_counter()
    oe = OracleEngine(wl, allr, alld, materialize=True)
    oe.run_workload()
    dt = time.perf_counter() - t0
    rows = len(oe.outputs)
    return {"value": rows / dt, "unit": "tokens/s", "cores": torch.get_num_threads(), "kind": "oracle",
            "sample": f"{desc}: {rows} attention rows (extend+decode) incl. tree ops, {dt:.1f} s"}, dt


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
    ap.add_argument("--workload", default="C3", choices=["C1", "C2", "C3", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary", default="C5", choices=["none", "C1", "C2", "C3", "C5"],
                    help="also time this workload (reported under 'secondary', context only)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        cpu, dt = run_oracle(args.workload)
        wl = make_workload(args.workload)
        line = {"impl": "reference", "metric": "attn tokens/s (extend+decode)", "value": cpu["value"],
                "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": dt * 1000.0, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{wl.name} (oracle sample)", "shape": f"{wl.shape.h_q}/{wl.shape.h_kv}/{wl.shape.head_dim}"},
                "cpu_baseline": cpu,
                "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

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

    from paper_2312_07104_b200.engine import Engine, plan_and_bank
    from paper_2312_07104_b200.tp import make_gather

    wl = make_workload(args.workload)
    gather = make_gather() if tp_path else None
    plan, bank = plan_and_bank(wl, dev, tp_rank=rank, tp_size=world)
    eng = Engine(wl, dev, tp_rank=rank, tp_size=world, gather=gather)
    tokens = plan.stats["extend_tokens"] + plan.stats["decode_tokens"]

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(max(2 * l2, 256 << 20), dtype=torch.uint8, device=dev)

    def barrier():
        if tp_path:
            dist.barrier()

    def step():
        eng.reset()
        eng.run_workload(bank)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    times = []
    eng.enable_timing(True)
    kern = {}
    tree_s = 0.0
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            eng.timer = []
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            barrier()
            times.append(a.elapsed_time(b))
            tree_s += eng.stats["tree_s"]
            for k_, v_ in eng.timing_summary().items():
                t = kern.setdefault(k_, [0.0, 0, 0, 0.0])
                for i in range(4):
                    t[i] += v_[i]
    launches = eng.stats["launches"]
    total_ms = sum(times)
    if tp_path:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = tokens * args.steps / (total_ms / 1000.0)

    peaks, peak_src = load_peaks()
    # dominant kernel by share of device time
    dom = max(kern.items(), key=lambda kv: kv[1][0])
    kind, (kms, knl, kcalls, kwork) = dom
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
    # this workload (profiles/r1_ncu_<kind>_traffic_<wl>.json, scripts/ncu_traffic.py), expressed for
    # this run's average launch: (captured DRAM bytes / captured algorithmic bytes) x algorithmic
    # bytes per launch here
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", f"r1_ncu_{kind}_traffic_{wl.name}.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj["traffic_over_algorithmic"] * (kwork / kcalls)
        traffic_src = {"file": os.path.relpath(tp, ROOT), "captured_launches": len(tj["launches"]),
                       "dram_bytes_per_captured_launch": tj["dram_bytes_per_launch"],
                       "algorithmic_bytes_per_captured_launch": tj["algorithmic_bytes_per_launch"],
                       "ratio": tj["traffic_over_algorithmic"]}
    # SURVEY §8(d) "always report both" denominators: the measured peak (frac) and the nominal one
    nominal = 2250.0 if kind == "extend" else 8000.0            # TFLOP/s dense bf16 | GB/s HBM3e
    roof.update({"achieved": achieved, "peak": peak, "frac": achieved / peak, "traffic": traffic,
                 "nominal_peak": nominal, "frac_nominal": achieved / nominal,
                 "traffic_source": traffic_src,
                 "peak_source": f"{peak_src} MEASURED_PEAKS.json" if peak_src == "measured" else "fallback",
                 "share_of_step": kms / total_ms if world == 1 else None})
    kernels = {k_: {"ms_per_step": v_[0] / args.steps, "calls_per_step": v_[2] // args.steps,
                    "launches_per_step": v_[1] // args.steps,
                    ("tflops" if k_ == "extend" else "gbs"): (v_[3] / (v_[0] / 1000.0) / (1e12 if k_ == "extend" else 1e9))}
               for k_, v_ in kern.items()}

    # ---------------------------------------------------------- e2e: host inputs, host outputs
    e2e = None
    if not args.no_e2e:
        from paper_2312_07104_b200.hostio import HostInputs, HostSink
        # every call's inputs live in pinned host memory and go host->device on a copy stream a few
        # calls ahead; every call's output lands in a preallocated pinned host buffer via a D2H
        # stream right after the call (paper_2312_07104_b200/hostio.py); sizes come from the plan
        hbank = HostInputs(bank, dev)
        h2d = hbank.h2d_bytes
        eng.enable_timing(False)
        hq = eng.hq * world
        sink = HostSink([torch.empty((len(c.hashes), hq, wl.shape.head_dim), dtype=torch.bfloat16, pin_memory=True)
                         for c in plan.calls], dev)
        d2h = [sink.d2h_bytes]
        eng.sink = sink
        for _ in range(args.warmup):            # untimed, like the device-resident steps
            sink.reset()
            hbank.reset()
            eng.reset()
            eng.run_workload(hbank)
            sink.join()
        torch.cuda.synchronize()
        e2e_times = []
        for it in range(max(1, args.steps)):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            sink.reset()
            a.record()
            hbank.reset()
            eng.reset()
            eng.run_workload(hbank)
            sink.join()
            b.record()
            torch.cuda.synchronize()
            e2e_times.append(a.elapsed_time(b))
        eng.sink = None
        e_ms = sum(e2e_times)
        if tp_path:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        e2e = {"value": tokens * len(e2e_times) / (e_ms / 1000.0), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h[0]),
               "ms_per_step": e_ms / len(e2e_times)}

    # ---------------------------------------------------------- secondary workload (context, same protocol)
    secondary = None
    if args.secondary != "none" and args.secondary != args.workload:
        del bank, eng
        torch.cuda.empty_cache()
        wl2 = make_workload(args.secondary)
        plan2, bank2 = plan_and_bank(wl2, dev, tp_rank=rank, tp_size=world)
        eng2 = Engine(wl2, dev, tp_rank=rank, tp_size=world, gather=gather)
        tok2 = plan2.stats["extend_tokens"] + plan2.stats["decode_tokens"]
        for _ in range(args.warmup):
            eng2.reset()
            eng2.run_workload(bank2)
        torch.cuda.synchronize()
        eng2.enable_timing(True)
        t2, kern2 = [], {}
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            eng2.timer = []
            a.record()
            eng2.reset()
            eng2.run_workload(bank2)
            b.record()
            torch.cuda.synchronize()
            barrier()
            t2.append(a.elapsed_time(b))
            for k_, v_ in eng2.timing_summary().items():
                t = kern2.setdefault(k_, [0.0, 0, 0, 0.0])
                for i in range(4):
                    t[i] += v_[i]
        ms2 = sum(t2)
        if tp_path:
            tt = torch.tensor([ms2], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms2 = float(tt.item())
        secondary = {
            "workload": wl2.name, "value": tok2 * len(t2) / (ms2 / 1000.0), "unit": "tokens/s",
            "ms_per_step": ms2 / len(t2), "tokens_per_step": tok2,
            "cache_hit_rate": plan2.stats["cached_prompt_tokens"] / max(1, plan2.stats["prompt_tokens"]),
            "kernels": {k_: {"ms_per_step": v_[0] / len(t2), "calls_per_step": v_[2] // len(t2),
                             ("tflops" if k_ == "extend" else "gbs_algorithmic"):
                                 v_[3] / (v_[0] / 1000.0) / (1e12 if k_ == "extend" else 1e9)}
                        for k_, v_ in kern2.items()},
            "note": "context only; decode of a shared 8k prefix uses rx_decode_cascade_append"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, _ = run_oracle(args.workload)

    if rank == 0:
        line = {
            "metric": "attn tokens/s (extend+decode), one attention layer",
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (rxgen: splitmix64 prefix-hash K/V/Q, mock-model tokens)",
            "config": {"workload": wl.name, "shape_hq_hkv_hd": [wl.shape.h_q, wl.shape.h_kv, wl.shape.head_dim],
                       "tokens_per_step": tokens, "extend_tokens": plan.stats["extend_tokens"],
                       "decode_tokens": plan.stats["decode_tokens"],
                       "cache_hit_rate": plan.stats["cached_prompt_tokens"] / max(1, plan.stats["prompt_tokens"]),
                       "parallelism": f"tp{world}" if world > 1 else ("tp1-selftest" if tp_path else "single"), "l2_flush": "2x L2 write before each timed step",
                       "num_slots": wl.num_slots},
            "gpu_launches": launches, "roofline": roof, "kernels": kernels,
            "tree_ms_per_step": tree_s * 1000.0 / args.steps,
            "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu, "secondary": secondary,
        }
        print(json.dumps(line))
    if tp_path:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
