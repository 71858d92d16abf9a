"""Build librx.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python paper_2312_07104_b200/build.py          # build if stale
    python paper_2312_07104_b200/build.py --force # rebuild everything
    python paper_2312_07104_b200/build.py --ptxas-v # print register / smem usage

Sources: csrc/host/*.cc (radix tree, pure host C++17) and csrc/kernels/*.cu
(sm_100a kernels + C-ABI wrappers).  Objects go to build/ next to this file.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build", "obj_" + os.path.basename(os.environ["RX_LIB_OUT"])) if os.environ.get("RX_LIB_OUT") \
    else os.path.join(HERE, "build")
LIB = os.environ.get("RX_LIB_OUT") or os.path.join(HERE, "librx.so")   # RX_LIB_OUT: A/B variant builds
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Wno-deprecated-gpu-targets", "-I", os.path.join(ROOT, "include")]
CU_FLAGS = ARCH + ["-lineinfo", "--expt-relaxed-constexpr"] + os.environ.get("RX_NVCC_FLAGS", "").split()


def _sources():
    out = []
    for sub in ("host", "kernels"):
        d = os.path.join(CSRC, sub)
        for f in sorted(os.listdir(d)):
            if f.endswith((".cc", ".cu")):
                out.append(os.path.join(d, f))
    return out


def _headers():
    hs = [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]
    for sub in ("host", "kernels"):
        d = os.path.join(CSRC, sub)
        hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".h", ".inc"))]
    return hs


def _compile(src, ptxas_v=False):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    cmd = [NVCC] + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += CU_FLAGS
        if ptxas_v:
            cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, ptxas_v: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    newest_in = max(os.path.getmtime(p) for p in srcs + _headers() + [__file__])
    if not force and not ptxas_v and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest_in:
        return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, ptxas_v), srcs))
    objs = [o for o, _ in results]
    if ptxas_v or verbose:
        for _, err in results:
            if err:
                sys.stderr.write(err)
    tmp = LIB + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, ptxas_v=a.ptxas_v, verbose=True))
