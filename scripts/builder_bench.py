"""The bench line's builder timings (bench.py `mask_builders`) on their own: c2 shape, flushed L2,
median of N steps (development aid).  python scripts/builder_bench.py [steps]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import masks as fmasks  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 9
cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
stream = torch.cuda.current_stream()
n, d, count = cfg.seq_len, cfg.head_dim, round(0.45 * cfg.seq_len)
for name, fn in (
        ("avg_query_threshold_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
            "avg_query_threshold", tau=1.0 / d), device_result=True)),
        ("avg_query_topk_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
            "avg_query_topk", top_k=count), device_result=True)),
        ("cached_threshold_ms", lambda: fmasks.build_mask_cached_qk(q, k, cfg, 0.5 / n, device_result=True))):
    fn()
    ts = sorted(bench.timed_steps(torch, fn, steps, flush, stream))
    print(f"{name}: median {ts[len(ts) // 2]:.4f} ms  min {ts[0]:.4f}", flush=True)
