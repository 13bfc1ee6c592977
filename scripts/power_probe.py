"""Run the c2 attention kernel back to back for ~2 s and sample SM clock / power / throttle
reasons with NVML (development aid: is the kernel power-capped?)."""
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
from paper_2509_16518_b200 import _lib  # noqa: E402

dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.45
B, H, N, D, M = 1, 12, 32760, 128, 128
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
shp = _lib.shape(B, H, N, D, M)


def run():
    _lib.call("fga_sparse_attn_fwd", q.data_ptr(), k.data_ptr(), v.data_ptr(), idx.data_ptr(), N, cnt.data_ptr(),
              o.data_ptr(), 0, None, shp, st)


pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd)))
        time.sleep(0.005)


for _ in range(5):
    run()
torch.cuda.synchronize()
th = threading.Thread(target=sampler)
th.start()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
n = 0
t0 = time.time()
while time.time() - t0 < 2.0:
    for _ in range(20):
        run()
    n += 20
    torch.cuda.synchronize()
b.record()
torch.cuda.synchronize()
stop.set()
th.join()
ms = a.elapsed_time(b) / n
s = sorted(samples)
clk = sorted(x[0] for x in samples)
pw = sorted(x[1] for x in samples)
reasons = 0
for x in samples:
    reasons |= x[2]
print(f"d={dens}: {ms:.3f} ms/launch back-to-back, SM clock median {clk[len(clk)//2]} MHz "
      f"(min {clk[0]}, max {clk[-1]}), power median {pw[len(pw)//2]:.0f} W max {pw[-1]:.0f} W, reasons 0x{reasons:x}")
