"""Raw pinned H2D bandwidth on this box (the ceiling of bench.py's e2e line)."""
import torch
n = 1478492160
x = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks in (1, 8, 16, 64):
    streams = [torch.cuda.Stream() for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    step = n // chunks
    for i in range(chunks):
        s = streams[i % 2]
        s.wait_event(e0)
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(x[i * step:(i + 1) * step], non_blocking=True)
    for s in streams:
        e1.wait(s) if False else None
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"chunks {chunks}: {n / ms / 1e6:.1f} GB/s")
