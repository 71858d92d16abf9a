#!/usr/bin/env bash
# Profiling recipe (run under gpurun on ONE GPU; see /opt/skills/guides/B200_PROFILING.md).
#   bash scripts/profile.sh [workload] [kernel-regex] [skip] [count]
# Writes to gpurun_out/:
#   launches_<wl>.csv   every launch of one bench step with its device time (cold-cache, serialised)
#   full_<wl>_<k>.ncu-rep   one `--set full` capture of the chosen kernel
set -u
WL=${1:-C3}
K=${2:-decode_kernel}
SKIP=${3:-20}
CNT=${4:-2}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# only this library's kernels (input generation launches thousands of small torch kernels)
timeout -k 5 2400 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k "regex:decode_kernel|decode_merge_kernel|cascade_merge_kernel|extend_kernel|extend_store_kernel|store_kv_kernel|tp_allgather_kernel" \
  --log-file gpurun_out/launches_${WL}.csv \
  python bench.py --workload "$WL" --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --configs none > gpurun_out/launches_${WL}.stdout 2>&1
timeout -k 5 900 $NCU --set full --clock-control none --import-source on -k "regex:${K}" -s ${SKIP} -c ${CNT} \
  -o gpurun_out/full_${WL}_${K} -f \
  python bench.py --workload "$WL" --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --configs none > gpurun_out/full_${WL}_${K}.stdout 2>&1
echo "profile done"
