"""Seeded random sweep of the device path against the oracle (GPU only).

Each case draws a shape (B, H, N, D, M incl. ragged last groups and M = 129..256 for the
shared-gather kernel), per-group list lengths (1 .. N, including full lists), a key pattern
(uniform random, contiguous runs, or the same list for every group of a head) and a scale, then
checks:
  * K1b compaction of the keep bytes and of the packed bits == np.nonzero (masks.py:75-91),
  * the fused selection (fga_select_compact) == the reference top-k / threshold rules
    (masks.py:131-147) on bf16 scores of the same rows,
  * sparse_attention == the chunked online softmax of sparse.py:138-155 within 2e-2,
  * the static tile stride and the dynamic longest-first scheduler give bitwise the same output.
Everything goes through libfgattn.so; the oracle is only the checker."""

import os

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
CASES = list(range(int(os.environ.get("FGA_FUZZ_CASES", "24"))))  # 200 in the round-2 stress run


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    b = int(rng.integers(1, 3))
    h = int(rng.integers(1, 4))
    n = int(rng.choice([97, 256, 700, 1000, 1537, 2048, 3001]))
    d = int(rng.choice([64, 128]))
    m = int(min(n, rng.choice([16, 64, 100, 128, 160, 256])))
    g = -(-n // m)
    pattern = ["random", "runs", "shared"][seed % 3]
    keep = np.zeros((b, h, g, n), np.uint8)
    for bb in range(b):
        for hh in range(h):
            shared = rng.random(n) < rng.uniform(0.05, 0.9)
            for gg in range(g):
                if pattern == "shared":
                    row = shared.copy()
                elif pattern == "runs":
                    row = np.zeros(n, bool)
                    for _ in range(int(rng.integers(1, 6))):
                        s0 = int(rng.integers(0, n))
                        row[s0: s0 + int(rng.integers(1, n // 3 + 2))] = True
                else:
                    row = rng.random(n) < rng.choice([0.01, 0.2, 0.5, 0.95, 1.0])
                if not row.any():
                    row[int(rng.integers(0, n))] = True
                keep[bb, hh, gg] = row
    scale = float(rng.choice([0.0, 0.05, 0.3]))  # 0: the default 1/sqrt(D)
    return b, h, n, d, m, keep, (scale or None)


@pytest.mark.parametrize("seed", CASES)
def test_fuzz_compaction_selection_attention(seed):
    b, h, n, d, m, keep, scale = _draw(seed)
    g = keep.shape[2]
    rows = b * h * g
    ref_lists = oracle.keep_to_lists(keep, np.zeros(keep.shape, np.float32))
    # K1b from bytes and from bits
    kd = torch.from_numpy(keep).cuda()
    dm = fga.compact_keep(kd, m, fill_sentinel=True)
    assert np.array_equal(dm.idx.cpu().numpy(), oracle.lists_to_padded(ref_lists, b, h, g, n)), seed
    dmb = fga.compact_keep_bits(fga.pack_keep_bits(kd), m, n)
    cnt = dmb.counts.cpu().numpy().reshape(-1)
    idxb = dmb.idx.cpu().numpy().reshape(rows, -1)
    assert all(np.array_equal(idxb[r, :cnt[r]], ref_lists[r]) for r in range(rows)), seed
    # fused selection on bf16 scores of the same rows
    rng = np.random.default_rng(seed)
    s16 = torch.from_numpy(rng.standard_normal((rows, n)).astype(np.float32) * 0.05).to(torch.bfloat16)
    x = s16.float().numpy()
    k_top = int(rng.integers(1, n + 1))
    idx = torch.empty((rows, n), dtype=torch.int32, device="cuda")
    c = torch.empty(rows, dtype=torch.int32, device="cuda")
    _lib.call("fga_select_compact", s16.cuda().data_ptr(), rows, n, _lib.FGA_SELECT_TOPK, 0.0, k_top, idx.data_ptr(),
              n, c.data_ptr(), 0, _stream())
    got = idx.cpu().numpy()
    for r in range(rows):
        want = np.sort(np.lexsort((np.arange(n), -x[r]))[:k_top])
        assert np.array_equal(got[r, :k_top], want), (seed, r)
    tau = float(np.quantile(x, 0.7))
    _lib.call("fga_select_compact", s16.cuda().data_ptr(), rows, n, _lib.FGA_SELECT_THRESHOLD, tau, 1, idx.data_ptr(),
              n, c.data_ptr(), 0, _stream())
    got, cc = idx.cpu().numpy(), c.cpu().numpy()
    for r in range(rows):
        want = np.flatnonzero(x[r] >= np.float32(tau))
        want = want if want.size else np.array([int(np.argmax(x[r]))])
        assert np.array_equal(got[r, :cc[r]], want), (seed, r)
    # attention vs the oracle, dynamic and static scheduling bitwise equal
    cfg = fga.AttnConfig(b, h, n, d, group_size=m, scale=scale, precision="bf16")
    q, k, v = (oracle.bf16_round(oracle.gaussian(cfg.dims, 10 * seed + i)) for i in range(3))
    qd, kd2, vd = (torch.from_numpy(t).cuda().to(torch.bfloat16) for t in (q, k, v))
    out = fga.sparse_attention(qd, kd2, vd, dm, cfg, out_dtype=torch.float32)
    ref = oracle.chunked_sparse_attention(q, k, v, ref_lists, m, cfg.scale, "bf16")
    err = float(np.abs(out.cpu().numpy() - ref).max())
    assert err <= ATOL, (seed, err)
    o_static = torch.empty_like(out)
    _lib.call("fga_sparse_attn_fwd_ex", qd.data_ptr(), kd2.data_ptr(), vd.data_ptr(), dm.idx.data_ptr(), dm.stride,
              dm.counts.data_ptr(), o_static.data_ptr(), _lib.FGA_OUT_F32, None,
              _lib.shape(*cfg.dims, m, cfg.scale), 0, -1, None, None, _lib.FGA_ATTN_STATIC, _stream())
    torch.cuda.synchronize()
    full = bool((dm.counts == n).all().item())
    if not full:  # (a full mask runs the dense kernel through sparse_attention)
        assert torch.equal(out, o_static), seed
