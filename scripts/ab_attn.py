"""Interleaved A/B timing of attention libraries at c2 (development aid).

    python scripts/ab_attn.py lib1.so lib2.so ...   (the in-tree libfgattn.so when none given)

Each library runs fga_sparse_attn_fwd (and, when exported, fga_sparse_attn_fwd_ex with the
static stride) on the same inputs; rounds alternate between libraries so box drift cancels."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402

libs = sys.argv[1:] or [_lib.LIB_PATH]
B, H, N, D, M = 1, 12, 32760, 128, 128
dens = 0.45
G = (N + M - 1) // M
st = torch.cuda.current_stream().cuda_stream
q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
count = round(dens * N)
keep = torch.empty(B * H * G, N, dtype=torch.uint8, device="cuda")
_lib.call("fga_random_keep", B * H * G, N, count, 7, keep.data_ptr(), st)
idx = torch.empty(B * H * G, N, dtype=torch.int32, device="cuda")
cnt = torch.empty(B * H * G, dtype=torch.int32, device="cuda")
_lib.call("fga_compact", keep.data_ptr(), None, B * H * G, N, idx.data_ptr(), N, cnt.data_ptr(), 0, st)
o = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
flops = 4 * D * M * count * H * G  # N = 255*128 + 120: close enough for A/B
P = ctypes.c_void_p
runs = []
for path in libs:
    lib = ctypes.CDLL(path)
    f = lib.fga_sparse_attn_fwd
    f.argtypes = [P, P, P, P, ctypes.c_int64, P, P, ctypes.c_int, P, _lib.FgaShape, P]
    sh = _lib.shape(B, H, N, D, M)
    runs.append((path + " fwd", lambda f=f, sh=sh: f(q.data_ptr(), k.data_ptr(), v.data_ptr(), idx.data_ptr(), N,
                                                    cnt.data_ptr(), o.data_ptr(), 0, None, sh, st)))
    if hasattr(lib, "fga_sparse_attn_fwd_ex"):
        fx = lib.fga_sparse_attn_fwd_ex
        fx.argtypes = [P, P, P, P, ctypes.c_int64, P, P, ctypes.c_int, P, _lib.FgaShape, ctypes.c_int64,
                       ctypes.c_int64, P, P, ctypes.c_int, P]
        runs.append((path + " static", lambda fx=fx, sh=sh: fx(q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                                idx.data_ptr(), N, cnt.data_ptr(), o.data_ptr(), 0,
                                                                None, sh, 0, -1, None, None, 4, st)))
times = {name: [] for name, _ in runs}
for rnd in range(6):
    for name, fn in runs:
        for _ in range(2):
            fn()
        for _ in range(5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = fn()
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, (name, rc)
            times[name].append(a.elapsed_time(b))
for name, ts in times.items():
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{name}: median {med:.3f} ms  min {ts[0]:.3f}  ({flops / med / 1e9:.0f} TF/s)", flush=True)
