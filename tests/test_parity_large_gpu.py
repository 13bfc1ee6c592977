"""Parity at the BASELINE.json Wan shapes (c3, c4, c5) and the c5 density-sweep endpoints.

The GPU computes the whole layer; the oracle (oracle.sparse_attention_group, the
chunked online softmax of /root/reference/pkg/src/sliceattn/sparse.py:138-155 +
tiled.py:48-77) recomputes sampled (head, group) units on the host, always
including the first group, a middle one and the last (short) group -- at c3/c5
N = 75600 = 590 * 128 + 80, so the last group has 80 rows and the 75600-key
rows take three compaction rounds.  Masks use the reference count rule
(max(1, round(d * N)) keys per group); the compacted lists are also checked
bit-exact against np.flatnonzero of the keep bytes.  Tolerance: 2e-2 max-abs
(BASELINE.json north_star).
"""

import numpy as np
import pytest

import oracle
from conftest import cuda_ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not cuda_ok():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402

ATOL = 2e-2


def _layer(heads, n, density, seed):
    cfg = fga.AttnConfig(1, heads, n, 128, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(seed)
    q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    count = max(1, round(density * n))
    keep = torch.empty((1, heads, cfg.num_groups, n), dtype=torch.uint8, device="cuda")
    _lib.call("fga_random_keep", heads * cfg.num_groups, n, count, seed, keep.data_ptr(),
              torch.cuda.current_stream().cuda_stream)
    mask = fga.compact_keep(keep, cfg.group_size)
    return cfg, q, k, v, keep, mask, count


def _check_units(cfg, q, k, v, keep, mask, count, out, units):
    worst = 0.0
    for h, gi in units:
        lo, hi = cfg.group_bounds(gi)
        c = int(mask.counts[0, h, gi])
        keys = mask.idx[0, h, gi, :c].cpu().numpy().astype(np.int64)
        assert c == count
        assert np.array_equal(keys, np.flatnonzero(keep[0, h, gi].cpu().numpy()))  # K1b bit-exact
        qh, kh, vh = (x[0, h].float().cpu().numpy() for x in (q, k, v))
        ref = oracle.sparse_attention_group(qh[lo:hi], kh, vh, keys, cfg.scale)
        got = out[0, h, lo:hi].float().cpu().numpy()
        worst = max(worst, float(np.abs(got - ref).max()))
    assert worst <= ATOL, worst
    return worst


@pytest.mark.parametrize("density", [0.1, 0.45, 0.9])
def test_c3_wan_720p_head(density):
    # c3 shape (12 heads at 720p), one head per density: the 80-row last group, 3-round rows
    cfg, q, k, v, keep, mask, count = _layer(1, 75600, density, seed=31)
    assert cfg.num_groups == 591 and cfg.group_bounds(590) == (75520, 75600)
    out = fga.sparse_attention(q, k, v, mask, cfg)
    _check_units(cfg, q, k, v, keep, mask, count, out, [(0, 0), (0, 1), (0, 295), (0, 589), (0, 590)])


def test_c4_wan14b_480p_forty_heads():
    cfg, q, k, v, keep, mask, count = _layer(40, 32760, 0.45, seed=41)
    out = fga.sparse_attention(q, k, v, mask, cfg)
    _check_units(cfg, q, k, v, keep, mask, count, out,
                 [(0, 0), (0, 255), (17, 128), (39, 0), (39, 255)])


@pytest.mark.parametrize("density", [0.1, 0.9])
def test_c5_wan14b_720p_sweep_endpoints(density):
    # c5: 40 heads at 720p, the ends of the 10-90% density sweep
    cfg, q, k, v, keep, mask, count = _layer(40, 75600, density, seed=51)
    out = fga.sparse_attention(q, k, v, mask, cfg)
    _check_units(cfg, q, k, v, keep, mask, count, out, [(0, 0), (0, 590), (21, 300), (39, 590)])


def test_c2_builder_mask_variable_lengths():
    # a mask from the device avg-query threshold builder (masks.py:121-150): list lengths vary
    # per group, so the dynamic longest-first scheduler reorders tiles; sampled groups vs oracle
    cfg = fga.AttnConfig(1, 2, 32760, 128, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    # per-group query scales spread the pooled scores, so the threshold keeps 10-50% of the keys
    f = torch.tensor([0.2 + 3.8 * (gi % 7) / 6 for gi in range(cfg.num_groups)], device="cuda")
    q = (q.float() * f.repeat_interleave(cfg.group_size)[: cfg.seq_len, None]).to(torch.bfloat16)
    mask = fga.build_mask(q, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1.02 / cfg.head_dim),
                          device_result=True)
    counts = mask.counts.cpu().numpy()
    assert counts.min() >= 1 and counts.max() > 2 * counts.min()
    out = fga.sparse_attention(q, k, v, mask, cfg)
    worst = 0.0
    for h, gi in [(0, 0), (0, int(counts[0, 0].argmax())), (1, int(counts[0, 1].argmin())), (1, 255)]:
        lo, hi = cfg.group_bounds(gi)
        keys = mask.keys_for(0, h, gi)
        ref = oracle.sparse_attention_group(*(x[0, h].float().cpu().numpy()[sl] for x, sl in
                                              ((q, slice(lo, hi)), (k, slice(None)), (v, slice(None)))),
                                            keys, cfg.scale)
        worst = max(worst, float(np.abs(out[0, h, lo:hi].float().cpu().numpy() - ref).max()))
    assert worst <= ATOL
