import torch, time
for mb in (1, 8, 8, 64, 512):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts2 = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    print(mb, "MB  isolated median %.3f ms (%.1f GB/s)   back-to-back %.3f ms each (%.1f GB/s)" % (
        sorted(ts)[5], (mb << 20) / sorted(ts)[5] / 1e6, a.elapsed_time(b) / 10, (mb << 20) / (a.elapsed_time(b) / 10) / 1e6))
