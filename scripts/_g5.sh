timeout 1500 python -m pytest tests -m gpu -x -q -k "extend_vs_oracle or json or chunked or host_io or mix" 2>&1 | tail -8 > gpurun_out/pytest_gpu_new.log
tail -4 gpurun_out/pytest_gpu_new.log
python scripts/pcie_bw.py > gpurun_out/pcie.txt 2>&1; cat gpurun_out/pcie.txt
timeout 900 python scripts/ablations.py fsm > gpurun_out/ablations_fsm.txt 2>&1; cat gpurun_out/ablations_fsm.txt
for M in 1 0; do RX_EXTEND_MULTI=$M timeout 600 python scripts/calls_timing.py JSON | tail -3; done > gpurun_out/calls_json2.txt 2>&1; cat gpurun_out/calls_json2.txt
