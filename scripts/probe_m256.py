"""Sparse attention with 129..256-row query groups: the shared-gather dual-tile kernel (default for
those shapes) vs the per-tile kernel (FGA_ATTN_KERNEL=ws), c2 shape (development aid)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402


def timeit(fn, flush, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 0.45
cfg = fga.AttnConfig(1, 12, 32760, 128, group_size=m, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
mask = fga.random_mask_device(cfg, dens, seed=1)
flops = fga.count_flops(cfg, mask).flops_matmul
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
res = {}
for name in ("dual", "ws"):
    os.environ["FGA_ATTN_KERNEL"] = name
    out = fga.sparse_attention(q, k, v, mask, cfg)
    res[name] = out.float()
    ms = timeit(lambda: fga.sparse_attention(q, k, v, mask, cfg), flush)
    print(f"M={m} d={dens} {name:4s} {ms:.3f} ms  {flops / ms / 1e9:.0f} TFLOP/s")
print("max |dual - ws|", float((res["dual"] - res["ws"]).abs().max()))
