"""HBM ceilings at the compaction's sizes: write-only (torch fill_) and copy (read+write) bandwidth for
buffers of the size K1b writes at c2 (~181 MB of lists), L2 flushed before every launch.

    python scripts/write_bw_probe.py"""
import torch

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def t_us(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


for mb in (64, 128, 181, 256, 403, 1024):
    n = mb * (1 << 20) // 4
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    y = torch.empty(n, dtype=torch.int32, device="cuda")
    med, mn = t_us(lambda: x.fill_(7))
    cm, cmn = t_us(lambda: y.copy_(x))
    by = n * 4
    print(f"{mb:5d} MB  write {med:7.1f} us {by / med / 1e3:7.0f} GB/s (best {by / mn / 1e3:.0f})   "
          f"copy {cm:7.1f} us {2 * by / cm / 1e3:7.0f} GB/s (best {2 * by / cmn / 1e3:.0f})", flush=True)
