"""fga_select_compact (top-k and threshold) on c2-shaped bf16 pooled scores (development aid / ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

H, N = 12, 32760
cfg = fga.AttnConfig(1, H, N, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
shp = _lib.shape(*cfg.dims, 128)
rows = H * cfg.num_groups
s16 = torch.empty((rows, N), dtype=torch.bfloat16, device="cuda")
ws = torch.empty(_lib.workspace_bytes(_lib.FGA_WS_POOLED_SCORES, shp), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
_lib.call("fga_pooled_scores_bf16", q.data_ptr(), k.data_ptr(), shp, s16.data_ptr(), ws.data_ptr(), ws.numel(), st)
idx = torch.empty((rows, N), dtype=torch.int32, device="cuda")
cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for mode, name in ((_lib.FGA_SELECT_TOPK, "top-k"), (_lib.FGA_SELECT_THRESHOLD, "threshold")):
    ts = []
    for _ in range(7):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.call("fga_select_compact", s16.data_ptr(), rows, N, mode, 1.0 / 128, int(0.45 * N), idx.data_ptr(), N,
                  cnt.data_ptr(), 0, st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"select {name}: median {sorted(ts)[3] * 1e3:.1f} us  (count mean {cnt.float().mean().item():.0f})")
