"""e2e (pinned host buffers -> GPU -> host) timing vs the number of head slabs (dev aid)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

cfg = fga.AttnConfig(1, 12, 32760, 128, precision="bf16")
st = torch.cuda.current_stream().cuda_stream
q, k, v = (torch.randn(cfg.dims, device="cuda").to(torch.bfloat16) for _ in range(3))
keep = torch.empty((1, 12, cfg.num_groups, cfg.seq_len), dtype=torch.uint8, device="cuda")
_lib.call("fga_random_keep", 12 * cfg.num_groups, cfg.seq_len, 14742, 77, keep.data_ptr(), st)
bits = fga.pack_keep_bits(keep)
hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
hb = bits.cpu().pin_memory()
ho = torch.empty(cfg.dims, dtype=torch.bfloat16).pin_memory()
for spec in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4", "6", "12"]):
    # "6u": uniform slabs; "5p4": 5 slabs, the one-head tail slab in 4 query-group runs
    base, _, parts = spec.rstrip("u").partition("p")
    slabs, tail, parts = int(base), not spec.endswith("u"), int(parts or 2)
    for _ in range(3):
        fga.sparse_attention_host(hq, hk, hv, hb, cfg, out=ho, slabs=slabs, tail=tail, tail_parts=parts)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fga.sparse_attention_host(hq, hk, hv, hb, cfg, out=ho, slabs=slabs, tail=tail, tail_parts=parts)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"slabs={spec}: e2e {ts[len(ts)//2]:.3f} ms (min {ts[0]:.3f})")
