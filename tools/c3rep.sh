for cap in 64 128 64 128; do GZ_BFS_CAP=$cap GZ_WATCHDOG_MS=100000 timeout 200 python tools/sweep_cfg.py C3 4 0 0 >> gpurun_out/c3rep.txt 2>&1; echo "cap $cap" >> gpurun_out/c3rep.txt; done
