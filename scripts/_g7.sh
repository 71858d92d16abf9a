timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 900 python scripts/e2e_probe.py C3 > gpurun_out/e2e_probe.txt 2>&1; cat gpurun_out/e2e_probe.txt
bash scripts/profile.sh C5 extend_kernel 0 2
/usr/local/cuda/bin/ncu -i gpurun_out/full_C5_extend_kernel.ncu-rep --page raw --csv > gpurun_out/full_C5_extend_raw.csv 2>&1
tail -3 gpurun_out/full_C5_extend_kernel.stdout
