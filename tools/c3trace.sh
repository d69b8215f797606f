# C3 convergence experiments (tail pulses per sweep, BFS depth); 60 s watchdog each
for cfg in "1000 272" "4000 272" "1000 512"; do
  set -- $cfg
  echo "== ktail $1 cap $2" >> gpurun_out/trace_c3b.txt
  GZ_KTAIL=$1 GZ_TAIL_AFTER=2 GZ_TRACE=1 GZ_WATCHDOG_MS=60000 timeout 200 python tools/sweep_cfg.py C3 4 $2 116 2>&1 | tail -6 >> gpurun_out/trace_c3b.txt
done
