for cfg in C3e C3q C1m128; do
  echo "== $cfg" >> gpurun_out/c3scale.txt
  GZ_WATCHDOG_MS=60000 timeout 200 python tools/sweep_cfg.py $cfg 4 -1,0 0 2>&1 | tail -3 >> gpurun_out/c3scale.txt
done
