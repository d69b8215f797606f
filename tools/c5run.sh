GZ_TRACE=1 GZ_WATCHDOG_MS=1800000 timeout 2300 python tools/c5_single.py > gpurun_out/c5_single_b.txt 2>&1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/c5_single_b.txt 2>&1
