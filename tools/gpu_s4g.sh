timeout 1200 python -m pytest tests/test_ozaki_gpu.py tests/test_streams_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider -x -k "not C5 and not c5" 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_drivers_gpu.py tests/test_reference_suite_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -3
BREAKDOWN=1 timeout 900 python tools/run_config.py C4 3 > gpurun_out/cfg_C4.log 2>&1; echo "C4 rc=$?"; grep -E "^  " gpurun_out/cfg_C4.log | head -6; tail -1 gpurun_out/cfg_C4.log | cut -c1-330
