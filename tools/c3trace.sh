GZ_TRACE=1 GZ_WATCHDOG_MS=150000 timeout 400 python tools/sweep_cfg.py C3 4 272 116 > gpurun_out/trace_c3a.txt 2>&1
