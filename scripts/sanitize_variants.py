"""Small launches of the variant attention kernels (pp, dual) for compute-sanitizer (development aid)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

for kern, m in [tuple(x.split(":")) for x in (sys.argv[1:] or ["pp:128", "dual:256"])]:
    m = int(m)
    os.environ["FGA_ATTN_KERNEL"] = kern
    cfg = fga.AttnConfig(1, 2, 1000, 128, group_size=m, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    mask = fga.random_mask_device(cfg, 0.4, seed=3)
    o = fga.sparse_attention(q, k, v, mask, cfg)
    torch.cuda.synchronize()
    print(kern, "ok", float(o.float().abs().max()))
