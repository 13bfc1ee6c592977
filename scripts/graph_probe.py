"""c1 (B=1, H=2, N=4096, D=64, d=0.3): per-call time of sparse_attention through the Python API
(eager: argument checks + ctypes launch each call) vs the same call captured once in a CUDA graph
and replayed (development aid / DESIGN.md evidence)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

cfg = fga.AttnConfig(1, 2, 4096, 64, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(3)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
mask = fga.random_mask_device(cfg, 0.3, seed=1)
for _ in range(20):
    fga.sparse_attention(q, k, v, mask, cfg)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    fga.sparse_attention(q, k, v, mask, cfg)
torch.cuda.synchronize()
eager_us = (time.perf_counter() - t0) / n * 1e6
graph = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    fga.sparse_attention(q, k, v, mask, cfg)
torch.cuda.current_stream().wait_stream(side)
with torch.cuda.graph(graph):
    for _ in range(10):
        out = fga.sparse_attention(q, k, v, mask, cfg)
graph.replay()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n // 10):
    graph.replay()
torch.cuda.synchronize()
graph_us = (time.perf_counter() - t0) / n * 1e6
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
fga.sparse_attention(q, k, v, mask, cfg)
b.record()
torch.cuda.synchronize()
print(f"c1 sparse_attention: eager {eager_us:.1f} us/call, CUDA-graph replay {graph_us:.1f} us/call, "
      f"one launch on the device {a.elapsed_time(b) * 1e3:.1f} us")
