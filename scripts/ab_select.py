"""A/B of fga_select_compact across libraries on c2 avg-query bf16 scores (development aid).

    python scripts/ab_select.py lib1.so lib2.so ...

Scores: fga_pooled_scores_bf16 of random Q/K at c2 (12 heads x 256 groups x 32760 keys), built
with the in-tree library.  Each library runs top-k (k = 14742) and threshold (tau = the 0.55
quantile); outputs must agree bitwise with the first library's.  Flushed-L2 median / min."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

libs = sys.argv[1:] or [_lib.LIB_PATH]
cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
s16 = fga.pooled_query_scores(q, k, cfg).to(torch.bfloat16).contiguous()
rows, n = s16.numel() // cfg.seq_len, cfg.seq_len
tau = float(torch.quantile(s16.float().view(-1)[:: 97], 0.55))
st = torch.cuda.current_stream().cuda_stream
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
P = ctypes.c_void_p
outs = {}
times = {}
fns = []
for path in libs:
    lib = ctypes.CDLL(path)
    f = lib.fga_select_compact
    f.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_int64, P, ctypes.c_int64, P,
                  ctypes.c_int, P]
    for mode, name in ((_lib.FGA_SELECT_TOPK, "topk"), (_lib.FGA_SELECT_THRESHOLD, "thr")):
        idx = torch.full((rows, n), -7, dtype=torch.int32, device="cuda")
        cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
        fns.append((f"{path} {name}", name, idx, cnt,
                    lambda f=f, mode=mode, idx=idx, cnt=cnt: f(s16.data_ptr(), rows, n, mode, tau, 14742, idx.data_ptr(), n,
                                                               cnt.data_ptr(), 0, st)))
for rnd in range(5):
    for key, name, idx, cnt, fn in fns:
        for _ in range(2):
            assert fn() == 0
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            times.setdefault(key, []).append(a.elapsed_time(b))
for key, name, idx, cnt, fn in fns:
    c = cnt.clone()
    mask = torch.arange(n, device="cuda")[None, :] < c[:, None]
    got = torch.where(mask, idx, torch.full_like(idx, -1))
    if name in outs:
        same = torch.equal(outs[name][0], c) and torch.equal(outs[name][1], got)
    else:
        outs[name] = (c, got)
        same = True
    ts = sorted(times[key])
    print(f"{key}: median {ts[len(ts) // 2] * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us  same={same}", flush=True)
