"""Small launches of the round-2 kernels for compute-sanitizer (memcheck / racecheck / synccheck):
fused selection + compaction (top-k, threshold, ragged n, scalar and TMA-bulk loads), bf16 and fused
threshold pooled-score epilogues + compaction with the argmax fallback, the TMA-bulk pooled mean,
the gather ring probe, the single-call cached builder, validation, tile order + timed attention."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
for n in (1000, 1003):  # TMA-bulk row load / scalar row load
    s16 = (torch.rand((6, n), device="cuda") * 0.01).to(torch.bfloat16)
    idx = torch.empty((6, n), dtype=torch.int32, device="cuda")
    cnt = torch.empty(6, dtype=torch.int32, device="cuda")
    for mode, tau in ((_lib.FGA_SELECT_TOPK, 0.0), (_lib.FGA_SELECT_THRESHOLD, 0.005), (_lib.FGA_SELECT_THRESHOLD, 1.0)):
        _lib.call("fga_select_compact", s16.data_ptr(), 6, n, mode, tau, 300, idx.data_ptr(), n, cnt.data_ptr(), 1, st)
cfg = fga.AttnConfig(1, 2, 1000, 128, precision="bf16")
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
m1 = fga.build_mask_avg_query(q, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1.0 / 128), device_result=True)
m2 = fga.build_mask_avg_query(q, k, cfg, fga.MaskBuilderConfig("avg_query_topk", top_k=333), device_result=True)
m3 = fga.build_mask_avg_query(q, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1e9), device_result=True)
m4 = fga.build_mask_cached_qk(q, k, cfg, 2.0 / cfg.seq_len, device_result=True)
m1.validate()
o = fga.sparse_attention(q, k, v, m1, cfg)
kk = torch.randn(3000, 128, device="cuda").to(torch.bfloat16)
keys = torch.sort(torch.randperm(3000, device="cuda")[:333]).values.to(torch.int32)
ok = torch.empty((384, 128), device="cuda", dtype=torch.bfloat16)
ov = torch.empty_like(ok)
c1 = torch.tensor([333], dtype=torch.int32, device="cuda")
_lib.call("fga_gather_ring_probe", kk.data_ptr(), kk.data_ptr(), 3000, 128, keys.data_ptr(), 333, c1.data_ptr(),
          ok.data_ptr(), ov.data_ptr(), st)
buf = torch.zeros(2 * 148, dtype=torch.int64, device="cuda")
shp = _lib.shape(*cfg.dims, cfg.group_size, cfg.scale)
_lib.call("fga_sparse_attn_fwd_timed", q.data_ptr(), k.data_ptr(), v.data_ptr(), m2.idx.data_ptr(), m2.stride,
          m2.counts.data_ptr(), o.data_ptr(), 0, None, shp, 0, -1, m2.tile_order(cfg).data_ptr(), None, 0,
          buf.data_ptr(), buf.numel(), st)
torch.cuda.synchronize()
print("ok", int(m1.counts.sum()), int(m2.counts.sum()), int(m3.counts.sum()), int(m4.counts.sum()))
