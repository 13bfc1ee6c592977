"""One fga_cached_group_max at c2 (ncu target for the cached builder's passes)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import masks  # noqa: E402

cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
for _ in range(2):
    masks.cached_group_max(q, k, cfg)
torch.cuda.synchronize()
