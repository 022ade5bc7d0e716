echo default; timeout 300 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 4096,544 24576,512
timeout 600 python -m pytest tests/test_gepp_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
echo dsmem; RLRA_B200_LIB=$PWD/tools/vlib/dsmem.so timeout 300 python tools/time_getrf.py 20000,220 10000,220 20000,200 10000,200 4096,544 24576,512
RLRA_B200_LIB=$PWD/tools/vlib/dsmem.so timeout 600 python -m pytest tests/test_gepp_gpu.py -q -p no:cacheprovider -x 2>&1 | tail -2
