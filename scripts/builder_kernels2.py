"""One avg-query threshold and one top-k build at c2 (ncu launch-list target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
for _ in range(2):
    fga.build_mask(q, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1.0 / 128), device_result=True)
    fga.build_mask(q, k, cfg, fga.MaskBuilderConfig("avg_query_topk", top_k=14742), device_result=True)
torch.cuda.synchronize()
