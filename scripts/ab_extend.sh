#!/usr/bin/env bash
# A/B the extend kernel across prebuilt library variants (variants/librx_*.so).
#   bash scripts/ab_extend.sh variants/librx_a.so variants/librx_b.so ...
set -u
cd "$(dirname "$0")/.."
for L in "$@"; do
  echo "== $L"
  export RX_LIB_OVERRIDE=$PWD/$L
  K="timeout 120 python scripts/kbench.py extend"
  $K --h 32 8 128 --batch 256 --prefix 0 --ext 384 | tail -1
  $K --h 32 8 128 --batch 256 --prefix 2048 --ext 384 | tail -1
  $K --h 32 8 128 --batch 256 --prefix 2048 --ext 384 --scatter | tail -1
  $K --h 64 8 128 --batch 1 --prefix 0 --ext 8192 | tail -1
  $K --h 64 8 128 --batch 128 --prefix 8192 --ext 128 | tail -1
  $K --h 32 32 128 --batch 64 --prefix 1536 --ext 128 | tail -1
done
