"""Attention kernel at c2 (12 heads, N=32760, 14742 keys per group) with the same list lengths but
different key patterns: uniform random (the benchmark), one contiguous block per group (sequential
L2 reads), every group of a head the same random list (hot L2 lines), and the dense kernel.
Separates the L2 access pattern from the LDGSTS issue cost of the gather."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402

B, H, N, D, M = 1, 12, 32760, 128, 128
G = (N + M - 1) // M
count = 14742
st = torch.cuda.current_stream().cuda_stream
q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
rows = B * H * G
keep = torch.empty(rows, N, dtype=torch.uint8, device="cuda")
_lib.call("fga_random_keep", rows, N, count, 7, keep.data_ptr(), st)
idx_rand = torch.empty(rows, N, dtype=torch.int32, device="cuda")
cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
_lib.call("fga_compact", keep.data_ptr(), None, rows, N, idx_rand.data_ptr(), N, cnt.data_ptr(), 0, st)
g = torch.arange(rows, device="cuda") % G
start = ((g * 97) % (N - count)).to(torch.int32)
idx_block = (start[:, None] + torch.arange(N, device="cuda", dtype=torch.int32)[None, :]).clamp(max=N - 1).contiguous()
idx_same = idx_rand.view(H, G, N)[:, :1, :].expand(H, G, N).reshape(rows, N).contiguous()
shp = _lib.shape(B, H, N, D, M)


def run(idx):
    return lambda: _lib.call("fga_sparse_attn_fwd_ex", q.data_ptr(), k.data_ptr(), v.data_ptr(), idx.data_ptr(), N,
                             cnt.data_ptr(), o.data_ptr(), 0, None, shp, 0, -1, None, None, _lib.FGA_ATTN_STATIC, st)


dense = lambda: _lib.call("fga_dense_attn_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), 0, None, shp,
                          st)
runs = [("random lists", run(idx_rand), 1.0), ("contiguous block per group", run(idx_block), 1.0),
        ("same random list for every group of a head", run(idx_same), 1.0), ("dense (all keys, TMA boxes)", dense,
                                                                            N / count)]
res = {name: [] for name, _, _ in runs}
for _ in range(5):
    for name, fn, _ in runs:
        fn()
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            res[name].append(a.elapsed_time(b))
for name, _, scale in runs:
    t = sorted(res[name])
    print(f"{name:45s} min {t[0]:.3f} ms  median {t[len(t) // 2]:.3f} ms  per-key-equivalent {t[0] / scale:.3f} ms")
