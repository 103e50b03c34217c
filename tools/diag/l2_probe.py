"""Does data written by one kernel stay in L2 for the next kernel?  Write a
buffer of `mb` MB (fill_), then read it (sum) — time the read right after the
write vs after a 256 MB flush (CUDA events, median of 20)."""
import torch


def t_read(buf, flush, after_flush):
    ts = []
    for _ in range(20):
        buf.fill_(1.0)
        if after_flush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        buf.sum()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[10]


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mb in (8, 16, 32, 48, 64, 96):
    buf = torch.empty((mb << 20) // 8, dtype=torch.float64, device="cuda")
    hot, cold = t_read(buf, flush, False), t_read(buf, flush, True)
    print(f"{mb:3d} MB: read after write {hot * 1e3:7.1f} us ({mb / 1024 / hot:.2f} TB/s), "
          f"after flush {cold * 1e3:7.1f} us ({mb / 1024 / cold:.2f} TB/s)")
