"""BASELINE.md §6 table rows from a committed bench log (dev tool): per config and phase, GPU tokens/s,
the fraction of the phase's roofline (extend: bf16 tensor, decode: HBM — measured peaks from the
bench line, nominal in brackets), and the oracle's tokens/s from scripts/oracle_rates.py output.

    python scripts/baseline_table.py profiles/r2_bench_v6_C3.log profiles/r2_oracle_rates.jsonl
"""
import json
import sys


def main(bench_log, oracle_jsonl):
    line = [x for x in open(bench_log) if x.startswith("{")][-1]
    d = json.loads(line)
    orc = {}
    for x in open(oracle_jsonl):
        r = json.loads(x)
        orc[r["config"]] = r
    recs = {"C3": d}
    recs.update(d.get("configs", {}))
    print("| Config | Phase | GPU tokens/s | Fraction of roofline | Oracle tokens/s |")
    print("|---|---|---|---|---|")
    for name in ("C3", "C1", "C2", "C4", "C5"):
        r = recs.get(name)
        if r is None:
            continue
        k = r["kernels"]
        o = orc.get(name, {})
        if name == "C3" and d.get("cpu_baseline"):
            o = {"tokens_per_s": d["cpu_baseline"]["value"], "cores": d["cpu_baseline"]["cores"]}
        e = k["extend"]
        print(f"| {name} | extend | {e['tokens_per_s'] / 1e6:.2f} M | {e['tflops']:.0f} TF/s = "
              f"{e['frac_bf16_measured']:.2f} of measured bf16 ({e['frac_bf16_nominal']:.2f} of 2.25 PF) | "
              f"{o.get('extend_tokens_per_s', float('nan')):.1f} |")
        c = k["decode"]
        print(f"| {name} | decode | {c['tokens_per_s'] / 1e6:.2f} M | {c['gbs']:.0f} GB/s unique = "
              f"{c['frac_hbm_measured']:.2f} of measured copy ({c['frac_hbm_nominal']:.2f} of 8 TB/s); "
              f"{c['gbs_logical']:.0f} GB/s logical | {o.get('decode_tokens_per_s', float('nan')):.1f} |")
        print(f"| {name} | extend+decode | **{r['value'] / 1e6:.2f} M** ({r['ms_per_step']:.2f} ms/pass) | — | "
              f"{o.get('tokens_per_s', float('nan')):.1f} ({o.get('cores', '?')} cores) |")


if __name__ == "__main__":
    main(*sys.argv[1:3])
