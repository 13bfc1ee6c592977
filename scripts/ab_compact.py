"""A/B of K1b compaction (fga_compact from keep bytes, fga_compact_bits from packed bits) across
library builds at c2 (3072 rows x 32760 keys, ~45 % kept); outputs must agree bitwise.

    python scripts/ab_compact.py lib1.so lib2.so ... [--dens 0.45] [--flush write|read]

--batch B times B back-to-back launches per event pair (no flush in between; the 181 MB of lists
exceed L2) -- the event clock ticks in ~2 us steps, too coarse for one 40 us launch.
--flush read evicts L2 by reading a 512 MiB buffer after writing it, so the timed kernel does not
start behind ~126 MB of dirty L2 lines from the flush (the default write flush leaves them)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
dens = float(sys.argv[sys.argv.index("--dens") + 1]) if "--dens" in sys.argv else 0.45
libs = [a for a in args if a.endswith(".so")] or [_lib.LIB_PATH]
n, rows = 32760, 12 * 256
gen = torch.Generator(device="cuda").manual_seed(0)
keep = (torch.rand((rows, n), device="cuda", generator=gen) < dens).to(torch.uint8)
bits = fga.pack_keep_bits(keep.view(1, 12, 256, n)).view(rows, -1).contiguous()
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
batch = int(sys.argv[sys.argv.index("--batch") + 1]) if "--batch" in sys.argv else 1
fmode = sys.argv[sys.argv.index("--flush") + 1] if "--flush" in sys.argv else "write"
fsum = torch.empty(1, dtype=torch.int64, device="cuda")


def do_flush():
    flush.zero_()
    if fmode == "read":
        torch.sum(flush.view(torch.int64), dim=0, out=fsum)
P, I64 = ctypes.c_void_p, ctypes.c_int64
fns, ref = [], {}
for path in libs:
    lib = ctypes.CDLL(path)
    fc, fb = lib.fga_compact, lib.fga_compact_bits
    fc.argtypes = [P, P, I64, I64, P, I64, P, ctypes.c_int, P]
    fb.argtypes = [P, I64, I64, P, I64, P, ctypes.c_int, P]
    for name in ("bytes", "bits"):
        idx = torch.empty((rows, n), dtype=torch.int32, device="cuda")
        cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
        if name == "bytes":
            fn = (lambda fc=fc, idx=idx, cnt=cnt: fc(keep.data_ptr(), None, rows, n, idx.data_ptr(), n, cnt.data_ptr(), 0, st))
        else:
            fn = (lambda fb=fb, idx=idx, cnt=cnt: fb(bits.data_ptr(), rows, n, idx.data_ptr(), n, cnt.data_ptr(), 0, st))
        fns.append((f"{path} {name}", name, idx, cnt, fn))
times = {}
for rnd in range(6):
    for key, name, idx, cnt, fn in fns:
        for _ in range(2):
            assert fn() == 0
        for _ in range(5):
            do_flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(batch):
                fn()
            b.record()
            torch.cuda.synchronize()
            times.setdefault(key, []).append(a.elapsed_time(b) / batch)
for key, name, idx, cnt, fn in fns:
    valid = torch.arange(n, device="cuda")[None, :] < cnt[:, None]
    got = torch.where(valid, idx, torch.full_like(idx, -1))
    same = True
    if name in ref:
        same = torch.equal(ref[name][0], cnt) and torch.equal(ref[name][1], got)
    else:
        ref[name] = (cnt.clone(), got)
    ts = sorted(times[key])
    print(f"{key}: median {ts[len(ts) // 2] * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us  same={same}", flush=True)
