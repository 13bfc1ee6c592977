"""K1b probe: fga_compact / fga_compact_bits at c2 (3072 rows x 32760 keys, ~45% kept).

Prints the median CUDA-event time and achieved GB/s of each (L2 flushed between steps).
Used with ncu: `ncu -k regex:compact --set full -c 2 python scripts/probe_compact.py`."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402


def main():
    n, g, h = 32760, 256, 12
    dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.45
    gen = torch.Generator(device="cuda").manual_seed(0)
    keep = (torch.rand((1, h, g, n), device="cuda", generator=gen) < dens).to(torch.uint8)
    bits = fga.pack_keep_bits(keep)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for name, fn, inb in (("bytes", lambda: fga.compact_keep(keep, 128), keep.numel()),
                          ("bits", lambda: fga.compact_keep_bits(bits, 128, n), bits.numel() * 4)):
        m = fn()
        live = 4 * int(m.counts.sum().item()) + 4 * m.counts.numel()
        ts = []
        for _ in range(9):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ts)[4]
        print(f"{name}: {ms * 1e3:.1f} us, {(inb + live) / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
