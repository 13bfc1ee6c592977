"""A/B of fga_cached_group_max across library builds at c2 (interleaved rounds, L2 flushed)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402

libs = sys.argv[1:] or [_lib.LIB_PATH]
B, H, N, D, M = 1, 12, 32760, 128, 128
G = (N + M - 1) // M
st = torch.cuda.current_stream().cuda_stream
q, k = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(2))
gmax = torch.empty(B, H, G, N, device="cuda")
sh = _lib.shape(B, H, N, D, M)
ws = torch.empty(_lib.workspace_bytes(_lib.FGA_WS_CACHED_GROUP_MAX, sh), dtype=torch.uint8, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.float32, device="cuda")
P = ctypes.c_void_p
fns = []
for path in libs:
    lib = ctypes.CDLL(path)
    f = lib.fga_cached_group_max
    f.argtypes = [P, P, _lib.FgaShape, ctypes.c_int, P, P, ctypes.c_size_t, P]
    fns.append((path, lambda f=f: f(q.data_ptr(), k.data_ptr(), sh, 1, gmax.data_ptr(), ws.data_ptr(), ws.numel(), st)))
times = {p: [] for p, _ in fns}
outs = {}
for rnd in range(4):
    for path, fn in fns:
        fn()
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = fn()
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, (path, rc)
            times[path].append(a.elapsed_time(b))
        outs[path] = gmax.clone()
ref = outs[libs[0]]
for path, ts in times.items():
    ts.sort()
    diff = (outs[path] != ref).float().mean().item()
    print(f"{path}: median {ts[len(ts) // 2]:.3f} ms  min {ts[0]:.3f}  (differs from the first build in {diff:.2e} of values)")
