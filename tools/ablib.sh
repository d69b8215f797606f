#!/bin/bash
# A/B two library builds (GZ_LIB_PATH): lone C1 seeds 0-7 and the bench, alternating.
# bash tools/ablib.sh A.so B.so tag [bench_reps]
a=$1; b=$2; tag=$3; reps=${4:-2}
out=gpurun_out
for r in $(seq 1 $reps); do
  for lib in $a $b; do
    n=$(basename $lib .so)
    GZ_LIB_PATH=$PWD/$lib timeout 300 python tools/lone_seeds.py "" > $out/ab_${tag}_lone_${n}_$r.txt 2>&1
    GZ_LIB_PATH=$PWD/$lib timeout 300 python bench.py --no-cpu-baseline --no-lone > $out/ab_${tag}_bench_${n}_$r.json 2>/dev/null
  done
done
for f in $out/ab_${tag}_*; do echo "$f: $(head -c 160 $f | tr '\n' ' ') ... $(grep -o '"value": [0-9.]*' $f | head -1)"; done
