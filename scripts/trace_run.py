"""Per-phase clock64 timeline of CTA 0's tile FGA_TRACE_IT (development aid; needs a trace build,
`_build.build_variant('trace', ['FGA_TRACE_ON=1'])`, run with FGA_LIB=build/variants/libtrace.so)."""
import os
import sys
import time

T0 = time.time()


def log(m):
    print(f"[{time.time() - T0:6.1f}s] {m}", flush=True)


# the library reads FGA_TRACE once (first launch), so it is set before any call; every call is
# traced and the last one's timeline is the file's content
os.environ["FGA_TRACE"] = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.txt"

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

log("imported torch")
dens = float(sys.argv[1]) if len(sys.argv) > 1 else 0.45
cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
q, k, v = (torch.randn(cfg.dims, device="cuda").to(torch.bfloat16) for _ in range(3))
dm = fga.random_mask_device(cfg, dens, seed=1)
torch.cuda.synchronize()
log("mask built")
for _ in range(3):
    fga.sparse_attention(q, k, v, dm, cfg)
    torch.cuda.synchronize()
    log("warm-up call done")
fga.sparse_attention(q, k, v, dm, cfg)
torch.cuda.synchronize()
log("traced call done")
