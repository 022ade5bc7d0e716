timeout 300 python tools/time_getrf.py 262144,512 262144,544 240000,512 > gpurun_out/tg_tall.txt 2>&1; cat gpurun_out/tg_tall.txt
timeout 900 python -m pytest tests/test_gepp_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -3
