"""A/B of the bf16 pooled-score pass (fga_pooled_scores_bf16, the top-k builder's score pass)
across library builds at c2: outputs compared bitwise with the first library's, flushed-L2 timing.
Q is scaled by 1, 6 and 20 so the scores also reach the exponent range's ends (huge / subnormal /
overflowing exp values).

    python scripts/ab_pooled16.py lib1.so lib2.so ..."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

libs = [a for a in sys.argv[1:] if a.endswith(".so")] or [_lib.LIB_PATH]
cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(3)
q0, k = (torch.randn(cfg.dims, device="cuda", generator=g) for _ in range(2))
k = k.to(torch.bfloat16)
shp = _lib.shape(*cfg.dims, cfg.group_size, cfg.scale)
ws = torch.empty(_lib.workspace_bytes(_lib.FGA_WS_POOLED_SCORES, shp, 1), dtype=torch.uint8, device="cuda")
out = torch.empty((cfg.heads * cfg.num_groups, cfg.seq_len), dtype=torch.int16, device="cuda")
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
P = ctypes.c_void_p
fns = []
for path in libs:
    lib = ctypes.CDLL(path)
    f = lib.fga_pooled_scores_bf16
    f.argtypes = [P, P, _lib.FgaShape, P, P, ctypes.c_size_t, P]
    fns.append((path, f))
for mult in (1.0, 6.0, 20.0):
    q = (q0 * mult).to(torch.bfloat16)
    ref, times = None, {}
    for rnd in range(4):
        for path, f in fns:
            for _ in range(5):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                rc = f(q.data_ptr(), k.data_ptr(), shp, out.data_ptr(), ws.data_ptr(), ws.numel(), st)
                b.record()
                torch.cuda.synchronize()
                assert rc == 0
                times.setdefault(path, []).append(a.elapsed_time(b) * 1e3)
            if rnd == 0:
                if ref is None:
                    ref = out.clone()
                    print(f"x{mult}: bf16 scores: {(ref == 0).float().mean():.3f} zero, "
                          f"{((ref & 0x7F80) == 0x7F80).float().mean():.4f} inf/nan", flush=True)
                else:
                    print(f"x{mult} {path}: bitwise equal {torch.equal(out, ref)} "
                          f"({(out != ref).sum().item()} differ)", flush=True)
    for path, ts in times.items():
        ts.sort()
        print(f"x{mult} {path}: median {ts[len(ts) // 2]:.1f} us  min {ts[0]:.1f} us", flush=True)
