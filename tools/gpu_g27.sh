timeout 900 python -m pytest tests/test_drivers_gpu.py -q -p no:cacheprovider -k "row_sharded_gepp or nccl" 2>&1 | tail -15
