"""Pinned host <-> device copy rates (development aid for the e2e pipeline)."""
import torch

n = 314 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(100 * 1024 * 1024, dtype=torch.uint8).pin_memory()
d2 = torch.empty(100 * 1024 * 1024, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"H2D 314 MB: {ms:.3f} ms = {n / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H 100 MB: {ms:.3f} ms = {100 * 1024 * 1024 / ms / 1e6:.1f} GB/s")


def both():
    ev = torch.cuda.current_stream().record_event()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


ms = t(both)
print(f"H2D 314 MB || D2H 100 MB: {ms:.3f} ms")
