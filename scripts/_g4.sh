timeout 1200 python -m pytest tests -m gpu -x -q -k "json or host_io" 2>&1 | tail -5 > gpurun_out/pytest_gpu_new.log
tail -3 gpurun_out/pytest_gpu_new.log
for C in 32 100000; do echo "== chunk $C"; RX_LAUNCH_CHUNK=$C timeout 600 python scripts/calls_timing.py C3 | tail -8; done > gpurun_out/calls_C3.txt 2>&1
cat gpurun_out/calls_C3.txt
timeout 600 python scripts/calls_timing.py JSON > gpurun_out/calls_json.txt 2>&1; tail -4 gpurun_out/calls_json.txt
timeout 900 python bench.py --secondary none > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
