"""Launch the cached builder a few times (for an ncu launch list of its kernels)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import masks  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 12
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32760
cfg = fga.AttnConfig(1, H, N, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
for _ in range(3):
    masks.cached_group_max(q, k, cfg)
torch.cuda.synchronize()
