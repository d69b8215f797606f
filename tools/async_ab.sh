for al in 1 2 4; do GZ_ASYNC_L=$al timeout 120 python tools/golden_check.py > gpurun_out/async_dbg_$al.txt 2>&1; done
GZ_ASYNC_L=2 timeout 300 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_async.log 2>&1
for al in 0 1 2 3 4; do GZ_ASYNC_L=$al GZ_PAIR_CONC=1 timeout 300 python tools/tail_knobs.py "12,0,96,4" > gpurun_out/async_knobs_$al.txt 2>&1; done
for al in 2 4; do GZ_ASYNC_L=$al timeout 100 python tools/big_configs.py C2 > gpurun_out/async_c2_$al.txt 2>&1; done
