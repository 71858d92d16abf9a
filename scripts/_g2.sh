bash scripts/ab_extend.sh variants/librx_085f9e7.so variants/librx_0d07bdd.so variants/librx_341feb7.so variants/librx_9d98b79.so variants/librx_bc64b8a.so > gpurun_out/ab_extend.txt 2>&1
bash scripts/profile.sh C3 decode_kernel
/usr/local/cuda/bin/ncu -i gpurun_out/full_C3_decode_kernel.ncu-rep --page raw --csv > gpurun_out/full_C3_decode_raw.csv 2>&1
ls -la gpurun_out
