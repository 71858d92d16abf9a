timeout 900 python scripts/e2e_probe.py C3 > gpurun_out/e2e_probe.txt 2>&1; cat gpurun_out/e2e_probe.txt
timeout 900 python scripts/ablations.py fsm > gpurun_out/ablations_fsm.txt 2>&1; cat gpurun_out/ablations_fsm.txt
