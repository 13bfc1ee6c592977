"""Static stride vs dynamic longest-first tile scheduling at c2 (development aid).

Uniform random mask (every group the same count) and a variable-length mask from the
avg-query threshold builder; median kernel time of sparse_attention, L2 flushed."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402


def timeit(fn, flush, iters=5):
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return ts


cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
masks = {"uniform_d0.45": fga.random_mask_device(cfg, 0.45, seed=1)}
f = torch.tensor([0.2 + 3.8 * (gi % 7) / 6 for gi in range(cfg.num_groups)], device="cuda")
qq = (q.float() * f.repeat_interleave(cfg.group_size)[: cfg.seq_len, None]).to(torch.bfloat16)
for tau in (1.02, 1.05):
    m = fga.build_mask(qq, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=tau / cfg.head_dim),
                       device_result=True)
    masks[f"avgq_thr{tau}"] = m
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
for name, m in masks.items():
    c = m.counts.float()
    flops = fga.count_flops(cfg, m).flops_matmul
    row = {"dynamic": [], "static": []}
    for rnd in range(6):   # interleaved rounds: power / clock drift hits both modes alike
        for mode in (("dynamic", "static") if rnd % 2 == 0 else ("static", "dynamic")):
            os.environ["FGA_ATTN_KERNEL"] = "" if mode == "dynamic" else "static"
            fga.sparse_attention(q, k, v, m, cfg)
            row[mode] += timeit(lambda: fga.sparse_attention(q, k, v, m, cfg), flush)
    out = []
    for mode, ts in row.items():
        ts.sort()
        out.append(f"{mode} median {ts[len(ts) // 2]:.3f} min {ts[0]:.3f} ms ({flops / ts[0] / 1e9:.0f} TF/s at min)")
    print(f"{name}: density {float(c.mean()) / cfg.seq_len:.3f} count cv {float(c.std() / c.mean()):.3f}  "
          + "  ".join(out), flush=True)
