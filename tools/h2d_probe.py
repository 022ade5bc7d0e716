"""Pinned host -> HBM copy bandwidth (the e2e path's floor): one copy, chunked
copies on one stream, chunked copies on two streams."""
import sys, time
import torch

dev = torch.device("cuda", 0)
nb = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_600_000_000
h = torch.empty(nb // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(nb // 8, dtype=torch.float64, device=dev)


def run(chunks, nstreams):
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    step = -(-h.numel() // chunks)
    for i, c0 in enumerate(range(0, h.numel(), step)):
        with torch.cuda.stream(streams[i % nstreams]):
            d[c0:c0 + step].copy_(h[c0:c0 + step], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return ms, nb / ms / 1e6


for chunks, ns in [(1, 1), (8, 1), (32, 1), (8, 2), (32, 2), (64, 4)]:
    run(chunks, ns)
    ms, gbs = run(chunks, ns)
    print(f"chunks {chunks:3d} streams {ns}: {ms:7.2f} ms  {gbs:6.1f} GB/s", flush=True)
# D2H of 48 MB (the factors)
x = torch.empty(6_000_000, dtype=torch.float64, device=dev)
hp = torch.empty(6_000_000, dtype=torch.float64, pin_memory=True)
hn = torch.empty(6_000_000, dtype=torch.float64)
for name, dst in [("pinned", hp), ("pageable", hn)]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        dst.copy_(x)
    torch.cuda.synchronize()
    print(f"D2H 48 MB {name}: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms")
