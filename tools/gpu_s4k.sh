timeout 900 python -m pytest tests/test_gepp_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 4096,544 24576,512 > gpurun_out/time_getrf_new.txt 2>&1; cat gpurun_out/time_getrf_new.txt
timeout 60 ./tools/lu_full_trace 10000 220 | tail -22
