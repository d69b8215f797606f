for al in 0 2 4; do GZ_ASYNC_L=$al timeout 300 python tools/sweep_cfg.py C3 4 0 0 > gpurun_out/c3async_$al.txt 2>&1; done
