#!/bin/bash
# Round-2 evidence session: GPU tests, smoke, bench (ours + reference arm),
# paper table, C2 timing.  Outputs under gpurun_out/ with the given tag.
tag=${1:-r2}
out=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $out/gpu_$tag.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -40 > $out/pytest_gpu_$tag.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err
timeout 600 python bench.py --impl reference > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
python tools/paper_table.py > $out/paper_table_$tag.txt 2>&1
python tools/lone_seeds.py "" > $out/lone_$tag.txt 2>&1
tail -3 $out/pytest_gpu_$tag.txt; cat $out/smoke_$tag.log | tail -2; tail -c 400 $out/bench_$tag.json; cat $out/paper_table_$tag.txt
