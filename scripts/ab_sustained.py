"""Sustained (power-capped) A/B of attention libraries at c2: each library runs back-to-back
launches of fga_sparse_attn_fwd for ~1.5 s (the board reaches its power cap), reporting ms per
launch and the median SM clock sampled through NVML during the run; libraries alternate with
1 s of idle between runs so each starts from the same thermal / power state.

    python scripts/ab_sustained.py lib1.so lib2.so ... [--rounds 3]"""
import ctypes
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402

args = [a for a in sys.argv[1:] if a.endswith(".so")] or [_lib.LIB_PATH]
rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
B, H, N, D, M = 1, 12, 32760, 128, 128
G = (N + M - 1) // M
st = torch.cuda.current_stream().cuda_stream
q, k, v = (torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
count = round(0.45 * N)
keep = torch.empty(B * H * G, N, dtype=torch.uint8, device="cuda")
_lib.call("fga_random_keep", B * H * G, N, count, 7, keep.data_ptr(), st)
idx = torch.empty(B * H * G, N, dtype=torch.int32, device="cuda")
cnt = torch.empty(B * H * G, dtype=torch.int32, device="cuda")
_lib.call("fga_compact", keep.data_ptr(), None, B * H * G, N, idx.data_ptr(), N, cnt.data_ptr(), 0, st)
o = torch.empty(B, H, N, D, device="cuda", dtype=torch.bfloat16)
flops = 4 * D * M * count * H * G
P = ctypes.c_void_p
try:
    import pynvml

    pynvml.nvmlInit()
    nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    nvh = None


def sample(stop, out):
    while not stop.is_set():
        if nvh is not None:
            out.append((pynvml.nvmlDeviceGetClockInfo(nvh, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(nvh) / 1000.0))
        time.sleep(0.02)


fns = []
for path in args:
    lib = ctypes.CDLL(path)
    f = lib.fga_sparse_attn_fwd
    f.argtypes = [P, P, P, P, ctypes.c_int64, P, P, ctypes.c_int, P, _lib.FgaShape, P]
    sh = _lib.shape(B, H, N, D, M)
    fns.append((path, lambda f=f, sh=sh: f(q.data_ptr(), k.data_ptr(), v.data_ptr(), idx.data_ptr(), N,
                                          cnt.data_ptr(), o.data_ptr(), 0, None, sh, st)))
res = {p: [] for p, _ in fns}
for _ in range(rounds):
    for path, fn in fns:
        torch.cuda.synchronize()
        time.sleep(1.0)
        fn()
        torch.cuda.synchronize()
        stop, smp = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, smp))
        th.start()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 600
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        ms = a.elapsed_time(b) / reps
        clk = sorted(c for c, _ in smp)[len(smp) // 2] if smp else -1
        pw = sorted(p for _, p in smp)[len(smp) // 2] if smp else -1
        res[path].append((ms, clk, pw))
for path, rs in res.items():
    ms = sorted(r[0] for r in rs)[len(rs) // 2]
    print(f"{path}: sustained {ms:.3f} ms/launch ({flops / ms / 1e9:.0f} TF/s)  runs "
          + " ".join(f"{r[0]:.3f}@{r[1]}MHz/{r[2]:.0f}W" for r in rs), flush=True)
