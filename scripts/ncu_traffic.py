"""DRAM traffic vs algorithmic bytes for the decode launches captured by ncu (profile.sh).

    python scripts/ncu_traffic.py gpurun_out/full_C3_decode_kernel.ncu-rep C3 --skip 20 > profiles/<name>.json

profile.sh captures `-k regex:decode_kernel -s SKIP -c N` of one bench step (the timed workload runs
first); in C3 every decode call is exactly one decode_kernel launch, so captured launch i is decode
call SKIP + i.  Algorithmic bytes of that call are recomputed on the host from the plan pass
(engine.decode_bytes: distinct pool rows x H_kv*hd*2*2 + q + o + slot indices).  bench.py reads the
result to fill roofline.traffic.  CPU only.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def ncu_launches(rep):
    out = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if "decode_kernel" not in d.get("Kernel Name", ""):
            continue

        def num(k, scale):
            return float(d[k].replace(",", "")) * scale
        units = rows[1][hdr.index("dram__bytes_read.sum")]
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units]
        unitw = rows[1][hdr.index("dram__bytes_write.sum")]
        scw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unitw]
        res.append({"kernel": d["Kernel Name"][:60], "dram_read": num("dram__bytes_read.sum", sc),
                    "dram_write": num("dram__bytes_write.sum", scw)})
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("workload", default="C3")
    ap.add_argument("--skip", type=int, default=20)
    a = ap.parse_args()
    from bench import make_workload
    from paper_2312_07104_b200.engine import Engine
    launches = ncu_launches(a.rep)
    want = {a.skip + i: i for i in range(len(launches))}
    wl = make_workload(a.workload)
    e = Engine(wl, plan_only=True)
    calls = [0]

    def hook(eng, slots, running, pos):
        k = calls[0]
        calls[0] += 1
        if k in want:
            alg, logical = eng.decode_bytes((slots, running, pos))
            launches[want[k]].update({"decode_call": k, "batch": int(len(running)),
                                      "algorithmic_bytes": alg, "logical_bytes": logical})
    e.on_decode_plan = hook
    e.run_workload()
    dram = sum(x["dram_read"] + x["dram_write"] for x in launches)
    alg = sum(x["algorithmic_bytes"] for x in launches)
    print(json.dumps({"source": os.path.basename(a.rep), "workload": a.workload, "launches": launches,
                      "dram_bytes_per_launch": dram / len(launches),
                      "algorithmic_bytes_per_launch": alg / len(launches),
                      "traffic_over_algorithmic": dram / alg}, indent=1))


if __name__ == "__main__":
    main()
