for cfg in "4294967296 16384" "8589934592 32768"; do set -- $cfg
RLRA_B200_SWEEP_BYTES=$1 RLRA_B200_SWEEP_PANEL=$2 BREAKDOWN=1 timeout 600 python tools/run_config.py C4 3 > gpurun_out/C4_$2.log 2>&1
echo bytes=$1 panel=$2; grep -E "sweep_oz|best_ms" gpurun_out/C4_$2.log | cut -c1-250
done
