# Every BASELINE config through tools/run_config.py (device-built inputs, CUDA-event timing, pivots digest, residual)
for c in C2 C3 C4 C5; do
  BREAKDOWN=1 timeout 900 python tools/run_config.py $c 3 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/cfg_$c.log | cut -c1-330
done
