"""Degenerate and malformed device masks behave like the reference (GPU only).

The reference raises ValueError for an empty group or an out-of-range key
(/root/reference/pkg/src/sliceattn/sparse.py:47-52) and NumericError for an
empty softmax denominator (tiled.py:75-76).  The device path checks a
DeviceIndexMask once on the device (fga_validate_mask) unless its producer
guarantees the invariants, the kernels flag violations in a status word
(FGA_ATTN_CHECK) and never read out of bounds, and the host pipeline raises
for an all-zero slice-mask row.  Also: the tile scheduler (dynamic,
longest-first order) gives bitwise the same outputs as the static stride.
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


def _qkv(cfg, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return tuple(torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))


def _mask(cfg, density=0.3, seed=1):
    return fga.random_mask_device(cfg, density, seed=seed)


def _copy(m, **kw):
    return fga.DeviceIndexMask(m.batch, m.heads, m.seq_len, m.group_size, kw.get("idx", m.idx.clone()),
                               kw.get("counts", m.counts.clone()))


CFG = dict(batch=1, heads=2, seq_len=1000, head_dim=64, group_size=128, precision="bf16")


def test_empty_group_raises_value_error():
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    m = _copy(_mask(cfg))
    m.counts[0, 1, 3] = 0
    with pytest.raises(ValueError, match="at least one key"):
        fga.sparse_attention(q, k, v, m, cfg)


def test_out_of_range_key_raises_value_error():
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    for bad in (cfg.seq_len, -5, 1 << 30):
        m = _copy(_mask(cfg))
        c = int(m.counts[0, 0, 2])
        m.idx[0, 0, 2, c - 1] = bad
        with pytest.raises(ValueError, match="out of range"):
            fga.sparse_attention(q, k, v, m, cfg)


def test_count_above_stride_and_unsorted_lists_are_rejected():
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    m = _copy(_mask(cfg))
    m.counts[0, 0, 0] = m.stride + 1
    with pytest.raises(fga.ShapeError):
        fga.sparse_attention(q, k, v, m, cfg)
    m = _copy(_mask(cfg))
    m.idx[0, 1, 4, :2] = m.idx[0, 1, 4, :2].flip(0)  # descending pair
    with pytest.raises(ValueError, match="sorted"):
        fga.sparse_attention(q, k, v, m, cfg)
    m = _copy(_mask(cfg))
    m.idx[0, 1, 5, 1] = m.idx[0, 1, 5, 0]  # duplicate key
    with pytest.raises(ValueError, match="sorted"):
        fga.sparse_attention(q, k, v, m, cfg)


def test_layout_contract_is_checked():
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    m = _mask(cfg)
    with pytest.raises(fga.ShapeError, match="int32"):
        fga.sparse_attention(q, k, v, _copy(m, idx=m.idx.to(torch.int64)), cfg)
    with pytest.raises(fga.ShapeError, match="contiguous"):
        wide = torch.zeros(m.idx.shape[:3] + (2 * m.stride,), dtype=torch.int32, device="cuda")
        wide[..., ::2] = m.idx
        fga.sparse_attention(q, k, v, _copy(m, idx=wide[..., ::2]), cfg)
    with pytest.raises(fga.ShapeError, match="counts"):
        fga.sparse_attention(q, k, v, _copy(m, counts=m.counts[:, :1].contiguous()), cfg)


def test_validated_masks_skip_the_check_and_compaction_without_scores_is_checked():
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    assert _mask(cfg).validated                       # exact-count device masks
    assert fga.random_mask(cfg, 0.2, seed=3).to_device().validated
    keep = torch.zeros((1, 2, cfg.num_groups, cfg.seq_len), dtype=torch.uint8, device="cuda")
    keep[..., ::7] = 1
    keep[0, 1, 2] = 0                                   # an empty row
    scores = torch.randn(keep.shape, device="cuda")
    m_fb = fga.compact_keep(keep, cfg.group_size, scores)  # argmax fallback: never empty
    assert m_fb.validated and int(m_fb.counts[0, 1, 2]) == 1
    fga.sparse_attention(q, k, v, m_fb, cfg)
    m_raw = fga.compact_keep(keep, cfg.group_size)       # no scores: the empty row stays empty
    assert not m_raw.validated
    with pytest.raises(ValueError, match="at least one key"):
        fga.sparse_attention(q, k, v, m_raw, cfg)
    bits = fga.pack_keep_bits(keep)
    with pytest.raises(ValueError):
        fga.sparse_attention(q, k, v, fga.compact_keep_bits(bits, cfg.group_size, cfg.seq_len), cfg)


def test_kernel_status_word_and_memory_safety():
    # fga_sparse_attn_fwd_ex: malformed rows are clamped (no out-of-bounds reads, the rest of the
    # layer is still right) and reported through the status word / FGA_ATTN_CHECK return codes
    cfg = fga.AttnConfig(**CFG)
    q, k, v = _qkv(cfg)
    m = _mask(cfg)
    good = fga.sparse_attention(q, k, v, m, cfg).float()
    bad = _copy(m)
    bad.idx[0, 0, 1, 0] = 1 << 30           # far outside K/V
    bad.counts[0, 1, 6] = 0
    status = torch.empty(2, dtype=torch.int32, device="cuda")
    o = torch.empty(cfg.dims, dtype=torch.bfloat16, device="cuda")
    for flags, want in ((_lib.FGA_ATTN_CHECK, _lib.FGA_EINVAL),
                        (_lib.FGA_ATTN_CHECK | _lib.FGA_ATTN_STATIC, _lib.FGA_EINVAL)):
        rc, msg = _lib.call_rc("fga_sparse_attn_fwd_ex", q.data_ptr(), k.data_ptr(), v.data_ptr(),
                               bad.idx.data_ptr(), bad.stride, bad.counts.data_ptr(), o.data_ptr(), _lib.FGA_OUT_BF16,
                               None, _lib.shape(*cfg.dims, cfg.group_size), 0, -1, None, status.data_ptr(), flags,
                               torch.cuda.current_stream().cuda_stream)
        assert rc == want and "at least one key" in msg
        bits = int(status[0])
        assert bits & _lib.FGA_STATUS_EMPTY and bits & _lib.FGA_STATUS_RANGE
    torch.cuda.synchronize()
    of = o.float()
    g = cfg.group_size
    keep_rows = torch.ones(cfg.dims[:3], dtype=torch.bool, device="cuda")
    keep_rows[0, 0, g:2 * g] = False
    keep_rows[0, 1, 6 * g:7 * g] = False
    assert torch.equal(of[keep_rows], good[keep_rows])            # untouched groups bitwise equal
    assert torch.isfinite(of).all() and (of[0, 1, 6 * g:7 * g] == 0).all()
    status.zero_()
    only_range = _copy(m)
    only_range.idx[0, 1, 0, 3] = -1
    rc, _ = _lib.call_rc("fga_sparse_attn_fwd_ex", q.data_ptr(), k.data_ptr(), v.data_ptr(),
                         only_range.idx.data_ptr(), only_range.stride, only_range.counts.data_ptr(), o.data_ptr(),
                         _lib.FGA_OUT_BF16, None, _lib.shape(*cfg.dims, cfg.group_size), 0, -1, None,
                         status.data_ptr(), _lib.FGA_ATTN_CHECK, torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.FGA_ERANGE


def test_host_pipeline_raises_on_an_empty_bits_row():
    cfg = fga.AttnConfig(1, 3, 777, 64, precision="bf16")
    q, k, v = (x.cpu().pin_memory() for x in _qkv(cfg))
    keep = torch.zeros((1, 3, cfg.num_groups, cfg.seq_len), dtype=torch.uint8, device="cuda")
    keep[..., 1::3] = 1
    bits = fga.pack_keep_bits(keep).cpu().pin_memory()
    out = fga.sparse_attention_host(q, k, v, bits, cfg)    # fine
    ref = fga.sparse_attention(*(x.cuda() for x in (q, k, v)), fga.compact_keep(keep, cfg.group_size), cfg)
    assert torch.equal(out, ref.cpu())
    bits[0, 2, 3] = 0
    with pytest.raises(ValueError, match="at least one key"):
        fga.sparse_attention_host(q, k, v, bits, cfg)


def test_import_padded_device_sorts_and_dedupes_like_the_host():
    rng = np.random.default_rng(8)
    b, h, n, m = 1, 2, 300, 64
    g = oracle.num_groups(n, m)
    pad = np.full((b, h, g, n), -1, np.int32)
    for r in range(b * h * g):
        c = int(rng.integers(1, 40))
        keys = rng.integers(0, n, size=c)             # unsorted, with duplicates
        pad.reshape(-1, n)[r, :c] = keys
    host = fga.import_padded(pad, m)
    dev = fga.import_padded(torch.from_numpy(pad).cuda(), m)
    assert dev.validated
    assert np.array_equal(fga.export_padded(host), fga.export_padded(dev).cpu().numpy())


def test_dynamic_longest_first_scheduler_is_bitwise_equal_to_static(monkeypatch):
    # variable list lengths (1 .. N keys) so the claim order differs from the tile order
    cfg = fga.AttnConfig(1, 3, 5000, 128, precision="bf16")
    q, k, v = _qkv(cfg, seed=4)
    rng = np.random.default_rng(2)
    lists = [np.sort(rng.choice(cfg.seq_len, size=int(rng.integers(1, cfg.seq_len)), replace=False))
             for _ in range(cfg.heads * cfg.num_groups)]
    mask = fga.SparseIndexMask._from_flat(1, cfg.heads, cfg.seq_len, cfg.group_size, lists)
    dyn = fga.sparse_attention(q, k, v, mask, cfg)
    monkeypatch.setenv("FGA_ATTN_KERNEL", "static")
    sta = fga.sparse_attention(q, k, v, mask, cfg)
    assert torch.equal(dyn, sta)
    # the longest-first order itself (fga_tile_order): per head, descending count, ties by group
    dm = mask.to_device()
    order = dm.tile_order(cfg).cpu().numpy()
    counts = dm.counts.cpu().numpy().reshape(cfg.heads, cfg.num_groups)
    want = np.concatenate([h * cfg.num_groups + np.lexsort((np.arange(cfg.num_groups), -counts[h]))
                           for h in range(cfg.heads)])
    assert np.array_equal(order, want)
    ref = oracle.masked_attention(*(x.float().cpu().numpy() for x in (q, k, v)), lists, cfg.group_size)
    assert np.abs(dyn.float().cpu().numpy() - ref).max() <= ATOL


def test_precision_full_is_refused_for_fp32_host_inputs():
    cfg = fga.AttnConfig(1, 1, 256, 64)  # precision='full' (the reference default)
    q, k, v = (fga.new_tensor(cfg, "gaussian", seed=s) for s in (1, 2, 3))
    with pytest.raises(NotImplementedError, match="precision='full'"):
        fga.sparse_attention(q, k, v, fga.full_mask(cfg), cfg)
    # bf16 CUDA tensors are already at the kernel's operand precision
    qd, kd, vd = (torch.from_numpy(x.data).cuda().to(torch.bfloat16) for x in (q, k, v))
    out = fga.sparse_attention(qd, kd, vd, fga.full_mask(cfg), cfg)
    ref = oracle.dense_attention(*(x.float().cpu().numpy() for x in (qd, kd, vd)))
    assert np.abs(out.float().cpu().numpy() - ref).max() <= ATOL
