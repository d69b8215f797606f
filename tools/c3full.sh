GZ_TRACE=1 GZ_WATCHDOG_MS=300000 timeout 500 python tools/sweep_cfg.py C3 4 -1 0 > gpurun_out/c3full.txt 2>&1
