"""Density / shape sweep on one GPU (development + evidence aid; bench.py is the contract line).

python scripts/sweep.py [configs] [densities]  ->  one JSON line per (config, density):
sparse layer latency (CUDA events, L2 flushed before each rep), effective TFLOP/s (4*D*pairs),
dense cuDNN SDPA latency on the same Q/K/V and the speedup."""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402  (CONFIGS)
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402


def timed(fn, flush, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    configs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2", "c3"]
    dens = [float(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0.2, 0.3, 0.45]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for cname in configs:
        heads, n, d, m, desc = bench.CONFIGS[cname]
        cfg = fga.AttnConfig(1, heads, n, d, group_size=m, precision="bf16")
        gen = torch.Generator(device="cuda").manual_seed(1234)
        q, k, v = (torch.randn(cfg.dims, device="cuda", generator=gen).to(torch.bfloat16) for _ in range(3))
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            t_dense = timed(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v), flush, 5)
        f_dense = 4 * d * heads * n * n
        for dd in dens:
            count = max(1, round(dd * n))
            keep = torch.empty((1, heads, cfg.num_groups, n), dtype=torch.uint8, device="cuda")
            _lib.call("fga_random_keep", heads * cfg.num_groups, n, count, 77, keep.data_ptr(), st)
            mask = fga.compact_keep(keep, m)
            del keep
            flops = fga.count_flops(cfg, mask).flops_matmul
            t = timed(lambda: fga.sparse_attention(q, k, v, mask, cfg), flush)
            print(json.dumps({"config": cname, "workload": desc, "density": dd, "keys_per_group": count,
                              "sparse_ms": round(t, 4), "tflops": round(flops / t / 1e9, 1),
                              "dense_cudnn_ms": round(t_dense, 4), "dense_tflops": round(f_dense / t_dense / 1e9, 1),
                              "speedup_vs_dense": round(t_dense / t, 3), "ideal_speedup": round(1 / dd, 3)}),
                  flush=True)
            del mask
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
