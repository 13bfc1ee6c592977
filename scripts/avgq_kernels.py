"""Launch the avg-query builders a few times (for an ncu launch list of their kernels)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 12
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32760
cfg = fga.AttnConfig(1, H, N, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
topk = fga.MaskBuilderConfig("avg_query_topk", top_k=int(0.45 * N))
thr = fga.MaskBuilderConfig("avg_query_threshold", tau=1.0 / 128)
for _ in range(2):
    fga.build_mask(q, k, cfg, topk, device_result=True)
    fga.build_mask(q, k, cfg, thr, device_result=True)
torch.cuda.synchronize()
