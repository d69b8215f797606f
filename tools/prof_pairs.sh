#!/bin/bash
# ncu evidence for the bench command at HEAD: the launch list (per-launch
# device times, cold-cache serialised) and one --set full capture of the
# batched gz_pairs_kernel launch (1184 C1 pairs, the bench's real regime).
tag=${1:-r2}
out=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-lone > $out/launches_$tag.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gz_pairs -s 6 -c 1 \
    -o $out/prof_$tag -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-lone > $out/prof_$tag.log 2>&1
ls -la $out/prof_$tag.ncu-rep $out/launches_$tag.csv
