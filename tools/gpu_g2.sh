timeout 900 python -m pytest tests/test_guard_gpu.py tests/test_ozaki_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_g2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_g2.log
tail -5 gpurun_out/pytest_g2.log
timeout 900 python bench.py > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; echo "bench rc=$?"
grep -E "Elapsed|Maximum resident" gpurun_out/bench_g2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_g2.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'] if d['e2e'] else None, d['parity'], json.dumps(d['C5']))"
CONFIG=C2 timeout 900 python tools/dist_bench_smoke.py > gpurun_out/dist_g2.json 2> gpurun_out/dist_g2.err; echo "dist rc=$?"
tail -c 1500 gpurun_out/dist_g2.json
