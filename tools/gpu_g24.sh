timeout 300 python tools/oz_prep_bench.py 2>&1 | tail -5
timeout 600 python bench.py --no-c5 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench_g24.json 2> gpurun_out/bench_g24.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_g24.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['other_kernels'])"
