"""Small K1b launches for compute-sanitizer: keep bytes with unaligned rows over several
rounds, empty rows (argmax fallback), the -1 tail; keep bits."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for n, m in ((1000, 128), (40001, 10000), (70003, 20000), (3000, 2)):  # (3000, 2): 3000 rows, persistent bits CTAs loop
    gr = -(-n // m)
    keep = (torch.rand((1, 2, gr, n), device="cuda", generator=g) < 0.4).to(torch.uint8)
    keep[0, 0, 1] = 0
    sc = torch.rand(keep.shape, device="cuda", generator=g)
    a = fga.compact_keep(keep, m, scores=sc, fill_sentinel=True)
    b = fga.compact_keep_bits(fga.pack_keep_bits(keep), m, n, fill_sentinel=True)
torch.cuda.synchronize()
print("ok", int(a.counts.sum()), int(b.counts.sum()))
