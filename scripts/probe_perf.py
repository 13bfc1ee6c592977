"""Quick kernel timing probe (development aid; bench.py is the contract)."""
import math
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402


def ptr(t):
    return t.data_ptr() if t is not None else None


def timeit(fn, iters=10, flush=None):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    B, H, N, D, M = 1, int(sys.argv[1]) if len(sys.argv) > 1 else 12, 32760, 128, 128
    for dens in ([float(sys.argv[2])] if len(sys.argv) > 2 else [0.45, 0.3, 0.2]):
        run(B, H, N, D, M, dens)


def run(B, H, N, D, M, dens):
    G = (N + M - 1) // M
    st = torch.cuda.current_stream().cuda_stream
    q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    count = round(dens * N)
    keep = torch.empty(B * H * G, N, dtype=torch.uint8, device="cuda")
    _lib.call("fga_random_keep", B * H * G, N, count, 7, ptr(keep), st)
    idx = torch.empty(B * H * G, N, dtype=torch.int32, device="cuda")
    cnt = torch.empty(B * H * G, dtype=torch.int32, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    o = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16)
    shp = _lib.shape(B, H, N, D, M)

    t_c = timeit(lambda: _lib.call("fga_compact", ptr(keep), None, B * H * G, N, ptr(idx), N, ptr(cnt), 0, st), flush=flush)
    t_s = timeit(lambda: _lib.call("fga_sparse_attn_fwd", ptr(q), ptr(k), ptr(v), ptr(idx), N, ptr(cnt), ptr(o),
                                   0, None, shp, st), flush=flush)
    t_d = timeit(lambda: _lib.call("fga_dense_attn_fwd", ptr(q), ptr(k), ptr(v), ptr(o), 0, None, shp, st), flush=flush)
    t_sdpa = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v), flush=flush)
    pairs = sum(min(M, N - g * M) for g in range(G)) * count * B * H
    f_s = 4 * D * pairs
    f_d = 4 * D * B * H * N * N
    print(f"compact {t_c:.3f} ms  {(B*H*G*N + 4*B*H*G*count)/t_c/1e6:.0f} GB/s")
    print(f"sparse  {t_s:.3f} ms  {f_s/t_s/1e9:.0f} TFLOP/s (d={dens})")
    print(f"dense(own) {t_d:.3f} ms  {f_d/t_d/1e9:.0f} TFLOP/s")
    print(f"sdpa    {t_sdpa:.3f} ms  {f_d/t_sdpa/1e9:.0f} TFLOP/s")
    print(f"speedup vs best dense: {min(t_d, t_sdpa)/t_s:.2f}x")
    prop = torch.cuda.get_device_properties(0)
    print(prop.name, prop.multi_processor_count, getattr(prop, "L2_cache_size", None))


if __name__ == "__main__":
    main()
