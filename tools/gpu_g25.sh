timeout 900 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c5 --breakdown > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1]); print(d['ms_per_step']); r=d['roofline']; print(json.dumps(r['other_kernels'])); print(r.get('int8_tensor'))"
head -20 gpurun_out/bench_c5.err
