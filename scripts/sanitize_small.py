"""Small launches of the production kernels for compute-sanitizer (development aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import masks  # noqa: E402

cfg = fga.AttnConfig(1, 2, 1000, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
masks.cached_group_max(q, k, cfg)
m = fga.random_mask_device(cfg, 0.4, seed=3)
o = fga.sparse_attention(q, k, v, m, cfg)
d = fga.flash_attention(q, k, v, cfg)
torch.cuda.synchronize()
print("ok", float(o.float().abs().max()), float(d.float().abs().max()))
