set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
K="timeout 120 python scripts/kbench.py extend"
( $K --h 32 8 128 --batch 256 --prefix 0 --ext 384 | tail -1
  $K --h 32 8 128 --batch 256 --prefix 2048 --ext 384 | tail -1
  $K --h 32 8 128 --batch 256 --prefix 2048 --ext 384 --scatter | tail -1
  $K --h 64 8 128 --batch 1 --prefix 0 --ext 8192 | tail -1
  $K --h 64 8 128 --batch 128 --prefix 8192 --ext 128 | tail -1
  $K --h 32 32 128 --batch 64 --prefix 1536 --ext 128 | tail -1 ) > gpurun_out/kbench_ext.txt 2>&1
cat gpurun_out/kbench_ext.txt
