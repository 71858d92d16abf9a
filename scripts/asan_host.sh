#!/usr/bin/env bash
# Build the HOST half of librx (radix tree + router, no CUDA) with ASan + UBSan
# and run the tree / router tests against it (CPU only).
#   bash scripts/asan_host.sh
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=/tmp/rx_asan
mkdir -p $OUT
g++ -O1 -g -std=c++17 -fPIC -shared -fsanitize=address,undefined -fno-omit-frame-pointer \
    -I "$ROOT/include" "$ROOT/paper_2312_07104_b200/csrc/host/radix_cache.cc" \
    "$ROOT/paper_2312_07104_b200/csrc/host/router.cc" "$ROOT/paper_2312_07104_b200/csrc/host/scheduler.cc" \
    "$ROOT/paper_2312_07104_b200/csrc/host/decode_steps.cc" -o $OUT/librx_host_asan.so
ASAN_LIB=$(g++ -print-file-name=libasan.so)
UBSAN_LIB=$(g++ -print-file-name=libubsan.so)
cd "$ROOT"
RX_LIB_OVERRIDE=$OUT/librx_host_asan.so LD_PRELOAD="$ASAN_LIB:$UBSAN_LIB" \
  ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
  python -m pytest tests/test_host_tree.py tests/test_router.py tests/test_theorem1.py tests/test_scheduler.py tests/test_engine_trace.py -q -p no:cacheprovider \
  -k "not exports"
