"""Fused selection + compaction (select.cu, fga_select_compact) and the single-call builders
(fga_build_mask_avgq / fga_build_mask_cached) against NumPy restatements of the reference:

  threshold: np.nonzero(s >= tau), empty -> [argmax(s)]   masks.py:75-91, 131-132
  top-k    : np.lexsort((arange(n), -s))[:k], ascending   masks.py:133-147, sparse.py:45-55

on bf16 score rows (the builders' analysis_scores rounding): heavy ties at the k-th value,
+-0, negative values, ragged n (not a multiple of 8 or 32), n up to the 75600 of c3/c5.
Bit-exact.  GPU only; every call goes through libfgattn.so."""

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


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _bf16_rows(rng, rows, n, distinct, signed=False):
    vals = rng.standard_normal(distinct).astype(np.float32)
    vals = vals if signed else np.abs(vals) * 0.01
    x = vals[rng.integers(0, distinct, size=(rows, n))]
    return torch.from_numpy(x).to(torch.bfloat16)  # RNE, like analysis_scores


def _select(s16, mode, tau=0.0, k=1, fill=0):
    rows, n = s16.shape
    d = s16.cuda().contiguous()
    idx = torch.full((rows, n), -7, dtype=torch.int32, device="cuda")
    cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
    _lib.call("fga_select_compact", d.data_ptr(), rows, n, mode, float(tau), int(k), idx.data_ptr(), n,
              cnt.data_ptr(), fill, _stream())
    torch.cuda.synchronize()
    return idx.cpu().numpy(), cnt.cpu().numpy()


def _ref_threshold(row, tau):
    keep = np.flatnonzero(row >= tau)
    return keep if keep.size else np.array([int(np.argmax(row))])


def _ref_topk(row, k):
    return np.sort(np.lexsort((np.arange(row.size), -row))[:k])


@pytest.mark.parametrize("n,distinct", [(1000, 5), (4093, 40), (32760, 300), (75600, 900), (75600, 3)])
def test_select_topk_bit_exact(n, distinct):
    rng = np.random.default_rng(n + distinct)
    s16 = _bf16_rows(rng, 8, n, distinct)
    x = s16.float().numpy()
    for k in (1, 37, n // 3, n // 2 + 7, n - 1, n):
        idx, cnt = _select(s16, _lib.FGA_SELECT_TOPK, k=k, fill=1)
        for r in range(x.shape[0]):
            ref = _ref_topk(x[r], k)
            assert cnt[r] == k
            assert np.array_equal(idx[r, :k], ref), (n, k, r)
            assert (idx[r, k:] == -1).all()


@pytest.mark.parametrize("n", [77, 1000, 32760, 75600])
def test_select_threshold_bit_exact_with_fallback(n):
    rng = np.random.default_rng(n)
    s16 = _bf16_rows(rng, 6, n, 200)
    x = s16.float().numpy()
    for tau in (float(np.quantile(x, 0.55)), float(x.max()) * 0.999, 1e9):
        idx, cnt = _select(s16, _lib.FGA_SELECT_THRESHOLD, tau=tau)
        for r in range(x.shape[0]):
            ref = _ref_threshold(x[r], np.float32(tau))
            assert cnt[r] == ref.size
            assert np.array_equal(idx[r, :ref.size], ref), (n, tau, r)


def test_select_signed_values_and_signed_zeros():
    # negative scores order below the positives; -0 and +0 tie (numpy compares values)
    rng = np.random.default_rng(3)
    n = 999
    s16 = _bf16_rows(rng, 4, n, 50, signed=True)
    bits = s16.view(torch.int16)
    bits[:, ::7] = 0
    bits[:, 3::11] = -32768  # -0.0
    x = s16.float().numpy()
    for k in (1, 100, 500, 998):
        idx, cnt = _select(s16, _lib.FGA_SELECT_TOPK, k=k)
        for r in range(4):
            assert np.array_equal(idx[r, :k], _ref_topk(x[r], k)), (k, r)
    idx, cnt = _select(s16, _lib.FGA_SELECT_THRESHOLD, tau=0.3)
    for r in range(4):
        ref = _ref_threshold(x[r], np.float32(0.3))
        assert np.array_equal(idx[r, :cnt[r]], ref)


def test_select_rejects_bad_arguments():
    s16 = torch.zeros((2, 100), dtype=torch.bfloat16)
    for k in (0, 101):
        with pytest.raises(fga.ShapeError):
            _select(s16, _lib.FGA_SELECT_TOPK, k=k)
    big = _lib.FGA_SELECT_MAX_N + 1
    rc, msg = _lib.call_rc("fga_select_compact", None, 1, big, _lib.FGA_SELECT_TOPK, 0.0, 1, None, big, None, 0,
                           _stream())
    assert rc != 0  # null pointers / too long a row are refused before any launch


def test_pooled_scores_bf16_equals_rounded_fp32():
    # the builders' bf16 score tensor is bitwise the rounded fp32 output of fga_pooled_scores
    for n, d, h, m in ((1000, 128, 2, 128), (640, 64, 3, 64), (4100, 128, 1, 128)):
        q = torch.randn(1, h, n, d, device="cuda").to(torch.bfloat16)
        k = torch.randn(1, h, n, d, device="cuda").to(torch.bfloat16)
        shp = _lib.shape(1, h, n, d, m)
        gc = -(-n // m)
        ws = torch.empty(_lib.workspace_bytes(_lib.FGA_WS_POOLED_SCORES, shp), dtype=torch.uint8, device="cuda")
        s32 = torch.empty((1, h, gc, n), device="cuda")
        s16 = torch.empty((1, h, gc, n), device="cuda", dtype=torch.bfloat16)
        _lib.call("fga_pooled_scores", q.data_ptr(), k.data_ptr(), shp, 1, s32.data_ptr(), ws.data_ptr(), ws.numel(),
                  _stream())
        _lib.call("fga_pooled_scores_bf16", q.data_ptr(), k.data_ptr(), shp, s16.data_ptr(), ws.data_ptr(),
                  ws.numel(), _stream())
        torch.cuda.synchronize()
        assert torch.equal(s16.float(), s32)


def test_workspace_too_small_is_refused():
    q = torch.randn(1, 1, 512, 64, device="cuda").to(torch.bfloat16)
    shp = _lib.shape(1, 1, 512, 64, 128)
    s = torch.empty((1, 1, 4, 512), device="cuda")
    ws = torch.empty(256, dtype=torch.uint8, device="cuda")
    with pytest.raises(fga.ShapeError, match="workspace"):
        _lib.call("fga_pooled_scores", q.data_ptr(), q.data_ptr(), shp, 1, s.data_ptr(), ws.data_ptr(), ws.numel(),
                  _stream())


@pytest.mark.parametrize("strategy", ["avg_query_threshold", "avg_query_topk"])
def test_build_mask_avgq_equals_selection_on_its_own_scores(strategy):
    # the single-call builder = the reference selection applied to fga_pooled_scores' (bf16) scores,
    # bit-exact, at a Wan-like row length (2 heads, N = 32760)
    cfg = fga.AttnConfig(1, 2, 32760, 128, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    scores = fga.pooled_query_scores(q, k, cfg).cpu().numpy()
    tau = float(np.quantile(scores, 0.6))
    b = fga.MaskBuilderConfig(strategy, tau=tau, top_k=9000)
    m = fga.build_mask_avg_query(q, k, cfg, b, device_result=True)
    counts = m.counts.cpu().numpy().reshape(-1)
    idx = m.idx.cpu().numpy().reshape(counts.size, -1)
    rows = scores.reshape(counts.size, -1)
    for r in range(0, counts.size, 37):
        ref = _ref_threshold(rows[r], np.float32(tau)) if strategy.endswith("threshold") else _ref_topk(rows[r], 9000)
        assert np.array_equal(idx[r, :counts[r]], ref), r


def test_build_mask_cached_single_call_equals_composition():
    cfg = fga.AttnConfig(1, 2, 2000, 128, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(9)
    q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    gmax = fga.cached_group_max(q, k, cfg).cpu().numpy()
    tau = 2.0 / cfg.seq_len
    m = fga.build_mask_cached_qk(q, k, cfg, tau, device_result=True)
    counts = m.counts.cpu().numpy().reshape(-1)
    idx = m.idx.cpu().numpy().reshape(counts.size, -1)
    rows = gmax.reshape(counts.size, -1)
    for r in range(counts.size):
        assert np.array_equal(idx[r, :counts[r]], _ref_threshold(rows[r], np.float32(tau))), r


@pytest.mark.parametrize("n,d,m", [(1000, 128, 128), (200, 64, 128), (4100, 128, 128), (1, 64, 1), (17, 128, 4),
                                   (40, 64, 40), (3000, 64, 2)])
def test_fused_threshold_builder_bits_and_fallback(n, d, m):
    # threshold decided in the pooled-score epilogue (keep bits + argmax fix-up, fga_build_mask_avgq):
    # bit-exact with the reference selection on the same (bf16) scores, ragged N, 30% of the groups
    # empty -> argmax fallback (masks.py:86-87); tiny N: the workspace covers the fused path;
    # (3000, 64, 2): 4500 rows, so the persistent bit-compaction CTAs loop over rows with fix-ups
    cfg = fga.AttnConfig(1, 3, n, d, group_size=m, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(n + d)
    q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    scores = fga.pooled_query_scores(q, k, cfg).cpu().numpy()
    rows = scores.reshape(-1, n)
    tau = float(np.quantile(rows.max(-1), 0.3)) * 1.0001
    m = fga.build_mask_avg_query(q, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=tau), device_result=True)
    counts = m.counts.cpu().numpy().reshape(-1)
    idx = m.idx.cpu().numpy().reshape(counts.size, -1)
    fallbacks = 0
    for r in range(counts.size):
        ref = _ref_threshold(rows[r], np.float32(tau))
        fallbacks += int((rows[r] >= np.float32(tau)).sum() == 0)
        assert np.array_equal(idx[r, :counts[r]], ref), r
    assert fallbacks > 0


def test_avg_query_builders_at_wan_shape_vs_oracle():
    # c2 row length (N = 32760, D = 128), one head: the GPU's pooled scores against the NumPy
    # restatement of masks.py:108-118 (mismatching bf16 scores counted and printed), and the
    # threshold / top-k lists against the reference selection on the reference's scores -- a key
    # may only differ where its score did (masks.py:131-147)
    n, d = 32760, 128
    cfg = fga.AttnConfig(1, 1, n, d, precision="bf16")
    q = oracle.bf16_round(oracle.gaussian(cfg.dims, 71))
    k = oracle.bf16_round(oracle.gaussian(cfg.dims, 72))
    ref = oracle.pooled_scores(q, k, cfg.group_size, None, "bf16").reshape(-1, n)
    got = fga.pooled_query_scores(torch.from_numpy(q).cuda().to(torch.bfloat16),
                                  torch.from_numpy(k).cuda().to(torch.bfloat16), cfg).cpu().numpy().reshape(-1, n)
    mism = got != ref
    print(f"pooled scores at N={n}: {mism.mean():.2e} of the bf16 values differ")
    assert mism.mean() < 2e-4
    tau = float(np.quantile(ref, 0.55))
    qd, kd = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (q, k))
    for b in (fga.MaskBuilderConfig("avg_query_threshold", tau=tau), fga.MaskBuilderConfig("avg_query_topk", top_k=14742)):
        m = fga.build_mask_avg_query(qd, kd, cfg, b, device_result=True)
        counts = m.counts.cpu().numpy().reshape(-1)
        idx = m.idx.cpu().numpy().reshape(counts.size, -1)
        for r in range(counts.size):
            want = _ref_threshold(ref[r], np.float32(tau)) if b.strategy.endswith("threshold") else _ref_topk(ref[r], 14742)
            have = idx[r, :counts[r]]
            if not np.array_equal(have, want):
                assert mism[r].any(), (b.strategy, r)   # only rows whose scores differ may differ
                flip = np.setxor1d(have, want)
                if b.strategy.endswith("threshold"):
                    assert mism[r, flip].all(), (b.strategy, r)  # and only at those keys


@pytest.mark.parametrize("mode", ["quantile", "bf16_value", "midpoint", "tiny", "huge"])
def test_fused_threshold_band_edges(mode, monkeypatch):
    # the fused threshold decides most scores by one accumulator compare (threshold_band in
    # maskbuild_tc.cu) and evaluates only a narrow band exactly: taus on a bf16 score value, on the
    # rounding midpoint between two bf16 values, and degenerate ones (tiny / huge: everything
    # exact) against the reference selection on the same scores, and against the all-exact
    # evaluation (FGA_THRESHOLD_EXACT=1) bit for bit
    n, d = 3000, 128
    cfg = fga.AttnConfig(1, 2, n, d, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(404)
    q, k = (torch.randn(cfg.dims, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    rows = fga.pooled_query_scores(q, k, cfg).cpu().numpy().reshape(-1, n)
    med = float(np.median(rows))
    b16 = np.array([med], np.float32).view(np.uint32)[0] >> 16
    val = float(np.array([b16 << 16], np.uint32).view(np.float32)[0])
    prev = float(np.array([(b16 - 1) << 16], np.uint32).view(np.float32)[0])
    tau = {"quantile": float(np.quantile(rows, 0.7)), "bf16_value": val, "midpoint": 0.5 * (val + prev),
           "tiny": 1e-30, "huge": 1e30}[mode]
    bc = fga.MaskBuilderConfig("avg_query_threshold", tau=tau)
    m = fga.build_mask_avg_query(q, k, cfg, bc, device_result=True)
    counts = m.counts.cpu().numpy().reshape(-1)
    idx = m.idx.cpu().numpy().reshape(counts.size, -1)
    for r in range(counts.size):
        assert np.array_equal(idx[r, :counts[r]], _ref_threshold(rows[r], np.float32(tau))), (mode, r)
    monkeypatch.setenv("FGA_THRESHOLD_EXACT", "1")
    me = fga.build_mask_avg_query(q, k, cfg, bc, device_result=True)
    assert torch.equal(me.counts, m.counts)
    assert all(torch.equal(me.idx.view(counts.size, -1)[r, :c], m.idx.view(counts.size, -1)[r, :c])
               for r, c in enumerate(counts.tolist()))


@pytest.mark.parametrize("gain", [8.0, 60.0])
def test_fused_threshold_extreme_scores(gain):
    # large query / key magnitudes: scores overflow to inf (kept when tau is finite) or underflow to
    # 0; the accumulator compare and the exact band must agree with the selection on the same scores
    n, d = 2000, 64
    cfg = fga.AttnConfig(1, 2, n, d, precision="bf16")
    g = torch.Generator(device="cuda").manual_seed(int(gain))
    q = (torch.randn(cfg.dims, device="cuda", generator=g) * gain).to(torch.bfloat16)
    k = (torch.randn(cfg.dims, device="cuda", generator=g) * gain).to(torch.bfloat16)
    rows = fga.pooled_query_scores(q, k, cfg).cpu().numpy().reshape(-1, n)
    finite = rows[np.isfinite(rows)]
    for tau in (float(np.quantile(finite, 0.5)) or 1e-3, 1e-30, 3.0e38):
        bc = fga.MaskBuilderConfig("avg_query_threshold", tau=tau)
        m = fga.build_mask_avg_query(q, k, cfg, bc, device_result=True)
        counts = m.counts.cpu().numpy().reshape(-1)
        idx = m.idx.cpu().numpy().reshape(counts.size, -1)
        for r in range(counts.size):
            assert np.array_equal(idx[r, :counts[r]], _ref_threshold(rows[r], np.float32(tau))), (gain, tau, r)
