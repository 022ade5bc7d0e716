timeout 900 python -m pytest tests/test_gepp_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python tools/time_getrf.py 16384,1024 16384,843 4096,544 4352,544 20000,512 12000,1000 24576,1024 > gpurun_out/tg_1024.txt 2>&1; cat gpurun_out/tg_1024.txt
RLRA_B200_LU_FULL=0 timeout 300 python tools/time_getrf.py 16384,1024 16384,843 4096,544 24576,1024 > gpurun_out/tg_1024b.txt 2>&1; cat gpurun_out/tg_1024b.txt
BREAKDOWN=1 timeout 900 python tools/run_config.py C3 3 > gpurun_out/cfg_C3.log 2>&1; echo "C3 rc=$?"; head -4 gpurun_out/cfg_C3.log; tail -1 gpurun_out/cfg_C3.log | cut -c1-200
