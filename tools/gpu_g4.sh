timeout 600 python -m pytest tests/test_drivers_gpu.py -q -p no:cacheprovider -k "nccl" > gpurun_out/pytest_g4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g4.log; tail -3 gpurun_out/pytest_g4.log
for c in C3 C4; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; tail -c 600 gpurun_out/bench_$c.json | head -c 600; echo
RLRA_B200_BENCH_DIST=1 RANK=0 WORLD_SIZE=1 LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-c5 > gpurun_out/dist_$c.json 2> gpurun_out/dist_$c.err; echo "dist $c rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/dist_$c.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity'])"
done
