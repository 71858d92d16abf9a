timeout 1200 python -m pytest tests -m gpu -x -q -k "mix or json" 2>&1 | tail -15 > gpurun_out/pytest_gpu_new.log
tail -3 gpurun_out/pytest_gpu_new.log
timeout 900 python scripts/ablations.py all > gpurun_out/ablations.txt 2> gpurun_out/ablations.err; cat gpurun_out/ablations.txt; tail -3 gpurun_out/ablations.err
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
