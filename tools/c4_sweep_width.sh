for w in 2048 4096 8192; do
  RLRA_B200_SWEEP_BYTES=4294967296 RLRA_B200_SWEEP_PANEL=$w BREAKDOWN=1 timeout 600 python tools/run_config.py C4 2 > gpurun_out/C4_$w.log 2>&1
  echo w=$w; grep -E "sweep_oz|best_ms" gpurun_out/C4_$w.log | cut -c1-160
done
