"""Run-to-run reproducibility of the dual-tile kernel at M = 256 (development aid)."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga
os.environ["FGA_ATTN_KERNEL"] = "dual"
cfg = fga.AttnConfig(1, 12, 32760, 128, group_size=256, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
m = fga.random_mask_device(cfg, 0.45, seed=1)
ref = fga.sparse_attention(q, k, v, m, cfg)
os.environ["FGA_ATTN_KERNEL"] = "ws"
ws = fga.sparse_attention(q, k, v, m, cfg)
os.environ["FGA_ATTN_KERNEL"] = "dual"
diff = 0
for _ in range(10):
    diff += int((fga.sparse_attention(q, k, v, m, cfg) != ref).sum())
print("dual rerun diffs:", diff, "max |dual-ws|", float((ref.float() - ws.float()).abs().max()))
