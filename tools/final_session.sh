#!/bin/bash
# End-of-round evidence: gpu tests, bench (+ reference arm), launch list, one full
# ncu capture of the solve kernel in the bench command, paper-table modes, C2.
tag=${1:-r1final}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$tag.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err
timeout 300 python tools/paper_table.py > gpurun_out/paper_table_$tag.txt 2>&1
timeout 200 python tools/big_configs.py C2 > gpurun_out/c2_$tag.txt 2>&1
(cd tools && timeout 300 python hier_breakdown.py) > gpurun_out/hier_$tag.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 3 --pairs 16 --no-cpu-baseline > gpurun_out/ncu_launch_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gz_tilesolve -s 48 -c 1 \
    -o gpurun_out/prof_$tag -f python bench.py --steps 1 --warmup 3 --pairs 16 --no-cpu-baseline > gpurun_out/ncu_full_$tag.log 2>&1
echo done
