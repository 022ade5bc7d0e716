timeout 300 python tools/time_getrf.py 262144,512 32768,544 4352,544 16384,1024 50000,720 > gpurun_out/tg_exact.txt 2>&1
cat > /tmp/tgf.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2002_07138_b200 import ops
dev = ops.check_device()
for m, n in [(262144,512),(32768,544),(4352,544),(16384,1024),(50000,720)]:
    a0 = torch.randn((n, m), dtype=torch.float64, device=dev).t()
    ts=[]
    for rep in range(4):
        a = ops.as_fmat(a0.clone()); torch.cuda.synchronize()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); p,_=ops.getrf_(a, exact=False); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    b = ops.as_fmat(a0.clone()); pe,_ = ops.getrf_(b)
    print(f"fast getrf {m} x {n}: {min(ts[1:])*1e3:9.1f} us  pivots equal to exact: {bool(torch.equal(p, pe))}")
PY
timeout 300 python /tmp/tgf.py > gpurun_out/tg_fast.txt 2>&1
paste gpurun_out/tg_exact.txt gpurun_out/tg_fast.txt
timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_drivers_gpu.py tests/test_gepp_gpu.py -q -p no:cacheprovider 2>&1 | tail -3
for c in C3 C4 C5; do BREAKDOWN=1 timeout 900 python tools/run_config.py $c 3 > gpurun_out/cfg_$c.log 2>&1; echo "$c rc=$?"; head -4 gpurun_out/cfg_$c.log; tail -1 gpurun_out/cfg_$c.log | cut -c1-200; done
