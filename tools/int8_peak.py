"""Dense int8 tensor-core peak of this B200, measured (not assumed 2 x bf16):
torch._int_mm (cuBLASLt int8 x int8 -> int32) on 8192^3, best of 10 (burst)
and back to back for 3 s (sustained), CUDA events.  Writes JSON to stdout."""
import json
import time

import torch

n = 8192
a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch._int_mm(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
ops = 2.0 * n ** 3
t0 = time.perf_counter()
cnt = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 3.0:
    for _ in range(20):
        torch._int_mm(a, b)
    cnt += 20
e1.record()
torch.cuda.synchronize()
sus = e0.elapsed_time(e1) / cnt
print(json.dumps({"int8_tops_burst": ops / (best / 1e3) / 1e12, "int8_tops_sustained": ops / (sus / 1e3) / 1e12,
                  "how": "torch._int_mm int8 8192^3 (cuBLASLt), 2*N^3 ops, best of 10 / back to back 3 s",
                  "gpu": torch.cuda.get_device_name(0)}))
