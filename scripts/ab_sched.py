"""A/B of attention libraries on a variable-length mask (development aid).

    python scripts/ab_sched.py lib1.so lib2.so ...

The mask is bench.py's variable-mask leg (avg-query threshold on Q scaled per group by 0.2..4.0,
c2), built once with the in-tree library; every library then runs fga_sparse_attn_fwd_timed with the
longest-first order (dynamic) and with the static stride.  Prints the flushed-L2 median / min and the
per-CTA tail fraction (longest CTA / mean CTA)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

libs = sys.argv[1:] or [_lib.LIB_PATH]
cfg = fga.AttnConfig(1, 12, 32760, 128, group_size=128)
st = torch.cuda.current_stream().cuda_stream
q, k, v = (torch.randn(*cfg.dims, device="cuda", dtype=torch.bfloat16) for _ in range(3))
f = torch.tensor([0.2 + 3.8 * (g % 7) / 6 for g in range(cfg.num_groups)], device="cuda")
qq = (q.float() * f.repeat_interleave(cfg.group_size)[: cfg.seq_len, None]).to(torch.bfloat16)
mask = fga.build_mask(qq, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1.02 / cfg.head_dim),
                      device_result=True)
flops = fga.count_flops(cfg, mask).flops_matmul
order = mask.tile_order(cfg)
o = torch.empty_like(q)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = torch.zeros(2 * sms, dtype=torch.int64, device="cuda")
P = ctypes.c_void_p
sh = _lib.shape(*cfg.dims, cfg.group_size, cfg.scale)
print(f"density {float(mask.counts.double().mean()) / cfg.seq_len:.3f}  cv "
      f"{float(mask.counts.double().std() / mask.counts.double().mean()):.3f}", flush=True)
runs = []
for path in libs:
    lib = ctypes.CDLL(path)
    ft = lib.fga_sparse_attn_fwd_timed
    ft.argtypes = [P, P, P, P, ctypes.c_int64, P, P, ctypes.c_int, P, _lib.FgaShape, ctypes.c_int64,
                   ctypes.c_int64, P, P, ctypes.c_int, P, ctypes.c_int64, P]
    for name, flags, od in (("dynamic", 0, order.data_ptr()), ("static", _lib.FGA_ATTN_STATIC, None)):
        def fn(ft=ft, flags=flags, od=od, b=None):
            return ft(q.data_ptr(), k.data_ptr(), v.data_ptr(), mask.idx.data_ptr(), mask.stride,
                      mask.counts.data_ptr(), o.data_ptr(), _lib.FGA_OUT_BF16, None, sh, 0, -1, od, None, flags,
                      b, buf.numel() if b else 0, st)
        runs.append((f"{path} {name}", fn))
times = {name: [] for name, _ in runs}
tails = {name: [] for name, _ in runs}
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
        flush.zero_()
        buf.zero_()
        assert fn(b=buf.data_ptr()) == 0
        torch.cuda.synchronize()
        t = buf.view(-1, 2).double()
        busy = (t[:, 1] - t[:, 0]) / 1e6
        tails[name].append(float(busy.max() / busy.mean()))
for name, ts in times.items():
    ts.sort()
    med = ts[len(ts) // 2]
    tl = sorted(tails[name])
    print(f"{name}: median {med:.3f} ms  min {ts[0]:.3f}  ({flops / med / 1e9:.0f} TF/s)  "
          f"tail {tl[len(tl) // 2]:.3f}", flush=True)
