timeout 1200 python -m pytest tests/test_ozaki_gpu.py tests/test_configs_gpu.py tests/test_drivers_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -8
BREAKDOWN=1 timeout 900 python tools/run_config.py C3 3 > gpurun_out/cfg_C3.log 2>&1; echo "C3 rc=$?"; grep -E "^  " gpurun_out/cfg_C3.log | head -14; tail -1 gpurun_out/cfg_C3.log | cut -c1-300
