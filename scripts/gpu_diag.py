"""Run each GPU kernel test in its own subprocess with a short timeout, so one
hang or fault cannot take the others down.  Prints one line per case.

    python scripts/gpu_diag.py [pytest -k expression] [--timeout S]
"""
import argparse
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    ap.add_argument("--file", default="tests/test_gpu_kernels.py")
    ap.add_argument("--timeout", type=int, default=120)
    a = ap.parse_args()
    col = subprocess.run([sys.executable, "-m", "pytest", a.file, "-m", "gpu", "--collect-only", "-q"] +
                         (["-k", a.k] if a.k else []), capture_output=True, text=True, cwd=ROOT)
    ids = [l.strip() for l in col.stdout.splitlines() if "::" in l]
    for tid in ids:
        try:
            r = subprocess.run([sys.executable, "-m", "pytest", tid, "-q", "-x", "-p", "no:cacheprovider"],
                               capture_output=True, text=True, cwd=ROOT, timeout=a.timeout)
            ok = r.returncode == 0
            msg = "" if ok else " | ".join([l for l in r.stdout.splitlines() if l.startswith("E ")][:4])[:600]
            print(f"{'PASS' if ok else 'FAIL'} {tid} {msg}", flush=True)
        except subprocess.TimeoutExpired:
            print(f"TIMEOUT {tid}", flush=True)


if __name__ == "__main__":
    main()
