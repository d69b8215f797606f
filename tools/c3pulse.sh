GZ_TRACE=2 timeout 300 python tools/sweep_cfg.py C3 4 0 0 > gpurun_out/c3pulse.txt 2>&1
