import torch, time
x = torch.empty(361*1024, dtype=torch.uint8).pin_memory()
d = torch.empty_like(x, device='cuda')
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for gap in (0, 100e-6):
    ts=[]; ws=[]
    for i in range(200):
        with torch.cuda.stream(s):
            e0.record(s); d.copy_(x, non_blocking=True); e1.record(s)
        t0=time.perf_counter(); s.synchronize(); ws.append(time.perf_counter()-t0)
        ts.append(e0.elapsed_time(e1)*1e3)
        if gap: time.sleep(gap)
    ts.sort(); ws.sort()
    print('gap', gap, 'H2D 361KB device us median', ts[100], 'p10', ts[20], 'host wait', ws[100]*1e6)
