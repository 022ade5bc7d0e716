timeout 600 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 262144,512 262144,544 32768,544 32768,512 4096,544 4352,544 16384,1024 16384,843 50000,720 > gpurun_out/time_getrf_r02.txt 2>&1; echo rc=$?
cat gpurun_out/time_getrf_r02.txt
