timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tail.log 2>&1
GZ_TRACE=2 GZ_PAIR_CONC=1 timeout 200 python tools/one_pair.py 2 8 > gpurun_out/trace_pulses_c1d.txt 2>&1
for tm in 0 1; do GZ_TAIL_MODE=$tm timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_tail$tm.json 2> gpurun_out/bench_tail$tm.err; done
GZ_PAIR_CONC=1 timeout 300 python tools/tail_knobs.py "12,0,96,4" > gpurun_out/tail_knobs3.txt 2>&1
