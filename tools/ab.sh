# A/B an env knob on the bench: bash tools/ab.sh VAR "v1 v2" tag
var=$1; vals=$2; tag=$3
for v in $vals; do for rep in 1 2; do env $var=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_${tag}_${v}_$rep.json 2>/dev/null; done; done
