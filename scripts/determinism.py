"""Run-to-run bitwise reproducibility of the attention output (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

cfg = fga.AttnConfig(1, int(sys.argv[1]) if len(sys.argv) > 1 else 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
m = fga.random_mask_device(cfg, 0.45, seed=1)
ref = fga.sparse_attention(q, k, v, m, cfg)
diff = 0
for _ in range(5):
    o = fga.sparse_attention(q, k, v, m, cfg)
    diff += int((o != ref).sum())
print("elements differing over 5 reruns:", diff)
