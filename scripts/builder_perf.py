"""Timing of the GPU mask builders at a Wan shape (development aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import masks  # noqa: E402


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


H = int(sys.argv[1]) if len(sys.argv) > 1 else 12
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32760
cfg = fga.AttnConfig(1, H, N, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
tau = 0.5 / N
print(f"H={H} N={N}")
print(f"cached_group_max       {timeit(lambda: masks.cached_group_max(q, k, cfg)):9.2f} ms")
print(f"build_mask_cached_qk   {timeit(lambda: fga.build_mask_cached_qk(q, k, cfg, tau, device_result=True)):9.2f} ms")
print(f"pooled_query_scores    {timeit(lambda: fga.pooled_query_scores(q, k, cfg)):9.2f} ms")
b = fga.MaskBuilderConfig("avg_query_topk", top_k=int(0.45 * N))
print(f"build_mask avgq top-k  {timeit(lambda: fga.build_mask(q, k, cfg, b, device_result=True)):9.2f} ms")
b = fga.MaskBuilderConfig("avg_query_threshold", tau=1.0 / 128)
print(f"build_mask avgq thr    {timeit(lambda: fga.build_mask(q, k, cfg, b, device_result=True)):9.2f} ms")
