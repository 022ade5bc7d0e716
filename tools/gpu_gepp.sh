RLRA_B200_LU_FULL=${RLRA_B200_LU_FULL:-1} timeout 900 python -m pytest tests/test_gepp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -15
