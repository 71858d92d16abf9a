#!/bin/bash
# Extend-kernel shape suite (scripts/kbench.py); pass RX_LIB_OVERRIDE=<.so> to time another build.
set -e
cd "$(dirname "$0")/.."
K="python scripts/kbench.py extend"
$K --h 64 8 128 --batch 1 --prefix 0 --ext 8192            # C5 root (8k causal)
$K --h 64 8 128 --batch 128 --prefix 8192 --ext 128 --shared-prefix   # C5 suffix over the shared 8k
$K --h 32 8 128 --batch 256 --prefix 2048 --ext 384        # C3 turn-3 shape, contiguous
$K --h 32 8 128 --batch 256 --prefix 2048 --ext 384 --ragged --half   # ... ragged, half fragmented
$K --h 32 8 128 --batch 256 --prefix 0 --ext 384           # C3 turn 0
$K --h 32 32 128 --batch 64 --prefix 1536 --ext 128 --shared-prefix   # C2 batch extend
$K --h 8 2 64 --batch 64 --prefix 1024 --ext 256           # hd 64
