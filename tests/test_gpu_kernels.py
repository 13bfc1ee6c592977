"""Kernel-level parity of libfgattn.so against the CPU oracle (GPU only).

Every call goes through the C ABI (ctypes) on torch-owned device memory.
Tolerances: indices/keep bits/gathered rows are bit-exact; attention outputs
<= 2e-2 max-abs vs the reference fp32 result (BASELINE.json north_star).
"""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_CASES, cuda_ok

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not cuda_ok():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_16518_b200 import _lib  # noqa: E402

ATOL = 2e-2


def ptr(t):
    return t.data_ptr() if t is not None else None


def stream():
    return torch.cuda.current_stream().cuda_stream


def workspace(op, shp):
    return torch.empty(max(_lib.workspace_bytes(op, shp), 1), dtype=torch.uint8, device="cuda")


def to_bf16_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda().to(torch.bfloat16)


def padded_dev(lists, b, h, n, m):
    g = oracle.num_groups(n, m)
    pad = oracle.lists_to_padded(lists, b, h, g, n)
    counts = (pad >= 0).sum(-1).astype(np.int32)
    return torch.from_numpy(pad).cuda(), torch.from_numpy(counts).cuda()


def tile_order(counts, b, h, n, d, m):
    tiles = b * h * (-(-n // m)) * (-(-m // 128))
    order = torch.empty(tiles, dtype=torch.int32, device="cuda")
    _lib.call("fga_tile_order", ptr(counts), _lib.shape(b, h, n, d, m), ptr(order), stream())
    return order


def run_sparse(q, k, v, idx, counts, b, h, n, d, m, scale=None, out_f32=True, lse=False):
    """fga_sparse_attn_fwd_ex with the FGA_ATTN_KERNEL selection (attn_kernel fixture); the
    dynamic scheduler claims tiles in fga_tile_order's longest-first order, with the kernel's
    status checks on (FGA_ATTN_CHECK)."""
    from paper_2509_16518_b200.sparse import attn_flags

    flags = attn_flags()
    order = None if flags & _lib.FGA_ATTN_STATIC else tile_order(counts, b, h, n, d, m)
    status = torch.empty(2, dtype=torch.int32, device="cuda")
    o = torch.empty((b, h, n, d), device="cuda", dtype=torch.float32 if out_f32 else torch.bfloat16)
    l = torch.empty((b, h, n), device="cuda", dtype=torch.float32) if lse else None
    _lib.call("fga_sparse_attn_fwd_ex", ptr(q), ptr(k), ptr(v), ptr(idx), idx.shape[-1], ptr(counts), ptr(o),
              _lib.FGA_OUT_F32 if out_f32 else _lib.FGA_OUT_BF16, ptr(l), _lib.shape(b, h, n, d, m, scale),
              0, -1, ptr(order), ptr(status), flags | _lib.FGA_ATTN_CHECK, stream())
    torch.cuda.synchronize()
    return o, l


# ------------------------------------------------------------------ K2 gather

@pytest.mark.parametrize("d", [64, 128, 192, 256])
@pytest.mark.parametrize("n_idx", [1, 5, 128, 300])
def test_gather_rows_bitwise(d, n_idx):
    g = torch.Generator().manual_seed(d + n_idx)
    mat = torch.randn(777, d, generator=g).to(torch.bfloat16).cuda()
    idx = torch.randint(0, 777, (n_idx,), generator=g, dtype=torch.int32)
    idx[: min(3, n_idx)] = 776  # duplicates + last row
    idx = idx.cuda()
    out = torch.empty(n_idx, d, dtype=torch.bfloat16, device="cuda")
    _lib.call("fga_gather_rows", ptr(mat), 777, d, ptr(idx), n_idx, ptr(out), stream())
    torch.cuda.synchronize()
    ref = mat[idx.long()]
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))


# ------------------------------------------------------------------ K1b compaction

@pytest.mark.parametrize("n", [33, 1000, 4096, 32760, 40001, 75600])
@pytest.mark.parametrize("fill", [0, 1])
def test_compact_bit_exact(n, fill):
    rng = np.random.default_rng(n)
    rows = 37
    keep = (rng.random((rows, n)) < rng.random((rows, 1))).astype(np.uint8)
    keep[3] = 0   # empty row -> argmax fallback
    keep[4] = 1   # full row
    keep[5] = 0
    keep[5, n - 1] = 7   # nonzero != 1 counts as kept
    scores = rng.standard_normal((rows, n)).astype(np.float32)
    scores[3, 11] = scores[3].max() + 1
    scores[3, 17] = scores[3, 11]   # tie -> first max (11)
    ref = oracle.lists_to_padded(oracle.keep_to_lists(keep, scores), 1, 1, rows, n)[0, 0]
    idx = torch.full((rows, n), 12345, dtype=torch.int32, device="cuda")
    cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
    kd = torch.from_numpy(keep).cuda()
    sd = torch.from_numpy(scores).cuda()
    _lib.call("fga_compact", ptr(kd), ptr(sd), rows, n, ptr(idx), n, ptr(cnt), fill, stream())
    torch.cuda.synchronize()
    got = idx.cpu().numpy()
    c = cnt.cpu().numpy()
    assert np.array_equal(c, (ref >= 0).sum(-1))
    if fill:
        assert np.array_equal(got, ref)
    else:
        for r in range(rows):
            assert np.array_equal(got[r, : c[r]], ref[r, : c[r]])
            assert (got[r, c[r]:] == 12345).all()


@pytest.mark.parametrize("n", [31, 1000, 32760, 40001])
@pytest.mark.parametrize("pad", [0, 1, 4])
@pytest.mark.parametrize("fill", [0, 1])
def test_compact_bits_strides(n, pad, fill):
    # bit-packed compaction into rows of stride n + pad: 16-byte aligned rows take the TMA bulk-store
    # flush (head / body / tail split at the output position mod 4), the others the per-key stores;
    # nothing is written past the count without the -1 fill, nothing past n with it
    rng = np.random.default_rng(n + pad)
    rows = 29
    keep = (rng.random((rows, n)) < rng.random((rows, 1))).astype(np.uint8)
    keep[2] = 0
    keep[3] = 1
    kd = torch.from_numpy(keep).cuda()
    words = (n + 31) // 32
    bits = torch.empty((rows, words), dtype=torch.int32, device="cuda")
    _lib.call("fga_pack_bits", ptr(kd), rows, n, ptr(bits), stream())
    stride = n + pad
    idx = torch.full((rows, stride), 12345, dtype=torch.int32, device="cuda")
    cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
    _lib.call("fga_compact_bits", ptr(bits), rows, n, ptr(idx), stride, ptr(cnt), fill, stream())
    torch.cuda.synchronize()
    got, c = idx.cpu().numpy(), cnt.cpu().numpy()
    for r in range(rows):
        pos = np.flatnonzero(keep[r])
        assert c[r] == pos.size, r
        assert np.array_equal(got[r, : c[r]], pos), r
        tail = got[r, c[r]:n]
        assert ((tail == -1) if fill else (tail == 12345)).all(), r
        assert (got[r, n:] == 12345).all(), r


def test_compact_unaligned_rows_without_scores():
    # row starts at odd byte offsets (n = 13) and no fallback: empty rows keep count 0
    rng = np.random.default_rng(1)
    keep = (rng.random((50, 13)) < 0.3).astype(np.uint8)
    keep[7] = 0
    idx = torch.zeros((50, 16), dtype=torch.int32, device="cuda")
    cnt = torch.empty(50, dtype=torch.int32, device="cuda")
    kd = torch.from_numpy(keep).cuda()
    _lib.call("fga_compact", ptr(kd), None, 50, 13, ptr(idx), 16, ptr(cnt), 1, stream())
    torch.cuda.synchronize()
    c = cnt.cpu().numpy()
    got = idx.cpu().numpy()
    for r in range(50):
        pos = np.flatnonzero(keep[r])
        assert c[r] == pos.size
        assert np.array_equal(got[r, : c[r]], pos)
        assert (got[r, c[r]:13] == -1).all()


# ------------------------------------------------------------------ K2+K3 attention

ATTN_CASES = [c for c in GOLDEN_CASES if c != "avgq_topk_ties"]


@pytest.fixture(params=["default", "ws", "static", "ws-static"])
def attn_kernel(request, monkeypatch):
    """The default dispatch (attn_ws.cu with the dynamic longest-first tile scheduler;
    attn_dual.cu for groups of 129..256 rows) and the FGA_ATTN_KERNEL selections: ws (attn_ws.cu
    for every shape), static (static tile stride), ws-static."""
    if request.param == "default":
        monkeypatch.delenv("FGA_ATTN_KERNEL", raising=False)
    else:
        monkeypatch.setenv("FGA_ATTN_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("name", ATTN_CASES)
@pytest.mark.parametrize("out_f32", [True, False])
def test_sparse_attention_matches_reference_golden(golden, name, out_f32, attn_kernel):
    g = golden(name)
    b, h, n, d = g.shape
    m = g.group_size
    q, k, v = (to_bf16_dev(oracle.bf16_round(t)) for t in (g.q, g.k, g.v))
    idx = torch.from_numpy(g["padded"].astype(np.int32)).cuda()
    cnt = torch.from_numpy(g["counts"].astype(np.int32)).cuda()
    o, lse = run_sparse(q, k, v, idx, cnt, b, h, n, d, m, g.cfg["scale"], out_f32, lse=True)
    ref = g["sparse_out"]
    err = np.abs(o.float().cpu().numpy() - ref).max()
    assert err <= ATOL, f"{name}: max-abs {err}"
    assert torch.isfinite(lse).all()


def test_sparse_attention_c1_error_is_small(golden):
    # tighter than the contract: fp32 out at c1 should sit near the bf16-P error (~1e-3)
    g = golden("c1_random30")
    b, h, n, d = g.shape
    q, k, v = (to_bf16_dev(oracle.bf16_round(t)) for t in (g.q, g.k, g.v))
    idx = torch.from_numpy(g["padded"].astype(np.int32)).cuda()
    cnt = torch.from_numpy(g["counts"].astype(np.int32)).cuda()
    o, _ = run_sparse(q, k, v, idx, cnt, b, h, n, d, 128, None, True)
    err = np.abs(o.cpu().numpy() - g["sparse_out"]).max()
    assert err <= 5e-3, err


def test_single_key_groups_copy_value_row():
    # a single listed key -> every output row equals v_j
    b, h, n, d, m = 1, 2, 512, 128, 128
    rng = np.random.default_rng(3)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    g = oracle.num_groups(n, m)
    lists = [np.array([int(rng.integers(n))]) for _ in range(b * h * g)]
    idx, cnt = padded_dev(lists, b, h, n, m)
    o, _ = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), idx, cnt, b, h, n, d, m)
    o = o.cpu().numpy()
    for r, lst in enumerate(lists):
        bb, hh, gg = r // (h * g), (r // g) % h, r % g
        # exact up to the 1-ulp error of the fused exp shift (l = 1 + O(2^-23))
        np.testing.assert_allclose(o[bb, hh, gg * m:(gg + 1) * m], np.broadcast_to(v[bb, hh, lst[0]], (m, d)),
                                   rtol=1e-6, atol=0)


@pytest.mark.parametrize("d", [64, 128])
def test_unsorted_duplicate_free_lists_and_stride(d, attn_kernel):
    # kernel consumes lists in the given order; result is order-independent
    b, h, n, m = 1, 1, 700, 128
    rng = np.random.default_rng(d)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    g = oracle.num_groups(n, m)
    lists = [np.sort(rng.choice(n, size=int(rng.integers(1, n)), replace=False)) for _ in range(g)]
    ref = oracle.masked_attention(q, k, v, lists, m)
    stride = n + 9
    pad = np.full((g, stride), -1, np.int32)
    counts = np.zeros(g, np.int32)
    for i, lst in enumerate(lists):
        perm = rng.permutation(lst)
        pad[i, : len(lst)] = perm
        counts[i] = len(lst)
    o, _ = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), torch.from_numpy(pad).cuda(),
                      torch.from_numpy(counts).cuda(), b, h, n, d, m)
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("order", ["ascending", "descending"])
@pytest.mark.parametrize("gain", [4.0, 16.0])
def test_online_rescale_large_dynamic_range(d, order, gain, attn_kernel):
    # Scores grow along the key list by ~50 (gain 4) or ~300 (gain 16) log2 units, so the
    # running max moves many times (the kernel's lazy-rescale slow path) -- or, descending,
    # never after the first chunk.
    b, h, n, m = 1, 2, 1536, 128
    rng = np.random.default_rng(11 + d)
    q = oracle.bf16_round(gain * rng.standard_normal((b, h, n, d)).astype(np.float32))
    ramp = (0.2 + 3.0 * np.arange(n) / n).astype(np.float32)
    k = oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32) * ramp[None, None, :, None])
    v = oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32))
    lists = oracle.random_lists(b, h, n, m, 0.6, seed=d)
    ref = oracle.masked_attention(q, k, v, lists, m)
    g = oracle.num_groups(n, m)
    pad = np.full((b * h * g, n), -1, np.int32)
    counts = np.zeros(b * h * g, np.int32)
    for i, lst in enumerate(lists):
        lst = np.asarray(lst)[::-1] if order == "descending" else np.asarray(lst)
        pad[i, : len(lst)] = lst
        counts[i] = len(lst)
    o, lse = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), torch.from_numpy(pad).cuda(),
                        torch.from_numpy(counts).cuda(), b, h, n, d, m, lse=True)
    assert np.isfinite(o.cpu().numpy()).all()
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL
    lse = lse.cpu().numpy()
    for i, lst in enumerate(lists):
        bb, hh, gg = i // (h * g), (i // g) % h, i % g
        lo, hi = gg * m, min(gg * m + m, n)
        sc = (q[bb, hh, lo:hi].astype(np.float64) @ k[bb, hh, lst].astype(np.float64).T) / np.sqrt(d)
        ref_l = np.log(np.exp(sc - sc.max(1, keepdims=True)).sum(1)) + sc.max(1)
        assert np.abs(lse[bb, hh, lo:hi] - ref_l).max() < 2e-2


@pytest.mark.parametrize("b,h,n,d", [(2, 3, 700, 128), (3, 2, 257, 64)])
def test_batched_heads(b, h, n, d, attn_kernel):
    # B > 1: tiles are numbered ((b*H + h)*G + g); every (b, h) reads only its own K/V rows
    m = 128
    rng = np.random.default_rng(b * 10 + d)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    lists = oracle.random_lists(b, h, n, m, 0.35, seed=b + d)
    ref = oracle.masked_attention(q, k, v, lists, m)
    idx, cnt = padded_dev(lists, b, h, n, m)
    o, _ = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), idx, cnt, b, h, n, d, m)
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL


@pytest.mark.parametrize("n,m", [(1, 1), (7, 7), (7, 1), (50, 50), (130, 3), (300, 300)])
def test_tiny_and_degenerate_shapes(n, m, attn_kernel):
    # single-row groups, one short tile, groups longer than a tile but shorter than two
    b, h, d = 1, 2, 64
    rng = np.random.default_rng(n * 31 + m)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    lists = oracle.random_lists(b, h, n, m, 0.5, seed=n + m)
    ref = oracle.masked_attention(q, k, v, lists, m)
    idx, cnt = padded_dev(lists, b, h, n, m)
    o, _ = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), idx, cnt, b, h, n, d, m)
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL


@pytest.mark.parametrize("m", [16, 64, 200, 256])
def test_group_sizes(m, attn_kernel):
    b, h, n, d = 1, 2, 600, 64
    rng = np.random.default_rng(m)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    lists = oracle.random_lists(b, h, n, m, 0.3, seed=m)
    ref = oracle.masked_attention(q, k, v, lists, m)
    idx, cnt = padded_dev(lists, b, h, n, m)
    o, _ = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), idx, cnt, b, h, n, d, m)
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL


@pytest.mark.parametrize("d,n", [(64, 1000), (128, 384)])
def test_dense_kernel_matches_dense_oracle(d, n):
    b, h = 1, 2
    rng = np.random.default_rng(n)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    ref = oracle.dense_attention(q, k, v)
    o = torch.empty((b, h, n, d), device="cuda", dtype=torch.float32)
    qd, kd, vd = to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v)  # keep alive across the launch
    _lib.call("fga_dense_attn_fwd", ptr(qd), ptr(kd), ptr(vd), ptr(o),
              _lib.FGA_OUT_F32, None, _lib.shape(b, h, n, d, 128), stream())
    torch.cuda.synchronize()
    assert np.abs(o.cpu().numpy() - ref).max() <= ATOL


def test_lse_matches_oracle():
    b, h, n, d, m = 1, 1, 256, 64, 128
    rng = np.random.default_rng(5)
    q, k, v = (oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32)) for _ in range(3))
    lists = oracle.random_lists(b, h, n, m, 0.5, seed=1)
    idx, cnt = padded_dev(lists, b, h, n, m)
    _, lse = run_sparse(to_bf16_dev(q), to_bf16_dev(k), to_bf16_dev(v), idx, cnt, b, h, n, d, m, lse=True)
    lse = lse.cpu().numpy()
    for gi, (lo, hi) in enumerate(oracle.group_ranges(n, m)):
        s = q[0, 0, lo:hi] @ k[0, 0, lists[gi]].T / np.sqrt(d)
        ref = np.log(np.exp(s - s.max(1, keepdims=True)).sum(1)) + s.max(1)
        assert np.abs(lse[0, 0, lo:hi] - ref).max() < 1e-3


# ------------------------------------------------------------------ K1a builders

def test_pooled_scores_and_threshold_keep(golden):
    g = golden("avgq_thr")
    b, h, n, d = g.shape
    m = g.group_size
    q, k = (to_bf16_dev(oracle.bf16_round(t)) for t in (g.q, g.k))
    gcount = oracle.num_groups(n, m)
    s = torch.empty((b, h, gcount, n), device="cuda", dtype=torch.float32)
    ws = workspace(_lib.FGA_WS_POOLED_SCORES, _lib.shape(b, h, n, d, m))
    _lib.call("fga_pooled_scores", ptr(q), ptr(k), _lib.shape(b, h, n, d, m), 1, ptr(s), ptr(ws), ws.numel(), stream())
    keep = torch.empty((b, h, gcount, n), device="cuda", dtype=torch.uint8)
    tau = float(g["tau"])
    _lib.call("fga_threshold_keep", ptr(s), s.numel(), tau, ptr(keep), stream())
    torch.cuda.synchronize()
    ref = g["scores"]
    got = s.cpu().numpy()
    # scores are bf16-rounded fp32 dot products: equal except at rare rounding boundaries
    mism = got != ref
    print(f"pooled scores (golden): {mism.mean():.2e} of the bf16 values differ")
    assert mism.sum() <= max(2, 1e-4 * mism.size)  # measured 0 here, 1.2e-5 at N = 32760
    assert np.abs(got - ref)[mism].max(initial=0) <= np.abs(ref).max() * 2 ** -7
    flips = (keep.cpu().numpy() != (ref >= tau))
    assert (flips <= mism).all()   # a keep bit can only flip where the score itself differs


@pytest.mark.parametrize("n,d,h,m", [(1000, 128, 2, 128), (640, 64, 3, 64), (4100, 128, 1, 128)])
def test_pooled_scores_tensor_cores_vs_oracle(n, d, h, m, monkeypatch):
    # q̄ split into three exact bf16 parts on the tensor cores (maskbuild_tc.cu pass 2) and the
    # CUDA-core tiles (FGA_POOLED_CC=1), both against the NumPy restatement of masks.py:108-118
    b = 1
    q = oracle.bf16_round(oracle.gaussian((b, h, n, d), 21))
    k = oracle.bf16_round(oracle.gaussian((b, h, n, d), 22))
    ref = oracle.pooled_scores(q, k, m, None, "bf16")
    gc = oracle.num_groups(n, m)
    qd, kd = to_bf16_dev(q), to_bf16_dev(k)
    for cc in ("0", "1"):
        monkeypatch.setenv("FGA_POOLED_CC", cc)
        s = torch.full((b, h, gc, n), -1.0, device="cuda", dtype=torch.float32)
        ws = workspace(_lib.FGA_WS_POOLED_SCORES, _lib.shape(b, h, n, d, m))
        _lib.call("fga_pooled_scores", ptr(qd), ptr(kd), _lib.shape(b, h, n, d, m), 1, ptr(s), ptr(ws), ws.numel(),
                  stream())
        torch.cuda.synchronize()
        got = s.cpu().numpy()
        mism = got != ref
        print(f"pooled scores n={n} d={d} cc={cc}: {mism.mean():.2e} of the bf16 values differ")
        assert mism.sum() <= max(2, 1e-4 * mism.size), (cc, mism.mean())
        assert np.abs(got - ref)[mism].max(initial=0) <= np.abs(ref).max() * 2 ** -7, cc


def test_topk_keep_matches_reference(golden):
    for name in ("avgq_thr", "avgq_topk_ties"):
        g = golden(name)
        scores = g["scores"]
        b, h, gc, n = scores.shape
        top_k = int(g["top_k"])
        sd = torch.from_numpy(scores).cuda()
        keep = torch.empty(scores.shape, dtype=torch.uint8, device="cuda")
        _lib.call("fga_topk_keep", ptr(sd), b * h * gc, n, top_k, ptr(keep), stream())
        torch.cuda.synchronize()
        lists = oracle.keep_to_lists(keep.cpu().numpy(), scores)
        ref = g.lists("topk_padded" if name == "avgq_thr" else "padded")
        assert all(np.array_equal(a, r) for a, r in zip(lists, ref)), name


def test_cached_group_max(golden):
    g = golden("cached_thr")
    b, h, n, d = g.shape
    m = g.group_size
    q, k = (to_bf16_dev(oracle.bf16_round(t)) for t in (g.q, g.k))
    gc = oracle.num_groups(n, m)
    gmax = torch.empty((b, h, gc, n), device="cuda", dtype=torch.float32)
    ws = workspace(_lib.FGA_WS_CACHED_GROUP_MAX, _lib.shape(b, h, n, d, m))
    _lib.call("fga_cached_group_max", ptr(q), ptr(k), _lib.shape(b, h, n, d, m), 1, ptr(gmax), ptr(ws), ws.numel(),
              stream())
    torch.cuda.synchronize()
    got = gmax.cpu().numpy()
    ref = g["gmax"]
    mism = got != ref
    print(f"cached group max (golden): {mism.mean():.2e} of the bf16 values differ")
    assert mism.sum() <= max(2, 1e-4 * mism.size)  # measured 1 value of 4096
    tau = float(g["tau"])
    flips = (got >= tau) != (ref >= tau)
    assert (flips <= mism).all()


@pytest.mark.parametrize("n,d,h", [(1000, 128, 2), (640, 64, 3), (200, 128, 1)])
def test_cached_group_max_tensor_cores_vs_oracle(n, d, h, monkeypatch):
    # ragged N (last group / key chunk partial), both head dims; the tensor-core passes
    # (maskbuild_tc.cu) and the CUDA-core passes (FGA_CACHED_CC=1) against the NumPy map
    m, b = 128, 1
    q = oracle.bf16_round(oracle.gaussian((b, h, n, d), 11))
    k = oracle.bf16_round(oracle.gaussian((b, h, n, d), 12))
    amap = oracle.attention_map(q, k, None, "bf16")
    tau = 2.0 / n
    keep_ref, ref = oracle.cached_keep(amap, m, tau, "bf16")
    gc = oracle.num_groups(n, m)
    qd, kd = to_bf16_dev(q), to_bf16_dev(k)
    for cc in ("0", "1"):
        monkeypatch.setenv("FGA_CACHED_CC", cc)
        gmax = torch.full((b, h, gc, n), -1.0, device="cuda", dtype=torch.float32)
        ws = workspace(_lib.FGA_WS_CACHED_GROUP_MAX, _lib.shape(b, h, n, d, m))
        _lib.call("fga_cached_group_max", ptr(qd), ptr(kd), _lib.shape(b, h, n, d, m), 1, ptr(gmax), ptr(ws),
                  ws.numel(), stream())
        torch.cuda.synchronize()
        got = gmax.cpu().numpy()
        mism = got != ref
        print(f"cached group max n={n} d={d} cc={cc}: {mism.mean():.2e} of the bf16 values differ")
        assert mism.sum() <= max(2, 1e-4 * mism.size), (cc, mism.mean())
        # where they differ, by one bf16 step at most
        if mism.any():
            rel = np.abs(got[mism] - ref[mism]) / np.maximum(np.abs(ref[mism]), 1e-30)
            assert rel.max() <= 2 ** -7, (cc, rel.max())
        flips = (got >= tau) != keep_ref
        assert (flips <= mism).all(), cc


def test_random_keep_exact_counts():
    rows, n, count = 64, 32760, 14742
    keep = torch.empty((rows, n), dtype=torch.uint8, device="cuda")
    _lib.call("fga_random_keep", rows, n, count, 1234, ptr(keep), stream())
    torch.cuda.synchronize()
    c = keep.sum(-1, dtype=torch.int64).cpu()
    assert (c == count).all()
    # rows differ from each other
    assert not torch.equal(keep[0], keep[1])


@pytest.mark.parametrize("n", [1024, 4000, 4096])
@pytest.mark.parametrize("cc", ["0", "1"])
def test_cached_group_max_tensor_cores_mismatch_rate_large(n, cc, monkeypatch):
    # up to 32 groups x 4096 keys per head: the fraction of bf16 group-max values that differ from
    # the NumPy map (printed with -s) stays below 1e-4, each by one bf16 step
    d, h, m = 128, 2, 128
    monkeypatch.setenv("FGA_CACHED_CC", cc)
    q = oracle.bf16_round(oracle.gaussian((1, h, n, d), 21))
    k = oracle.bf16_round(oracle.gaussian((1, h, n, d), 22))
    amap = oracle.attention_map(q, k, None, "bf16")
    keep_ref, ref = oracle.cached_keep(amap, m, 0.5 / n, "bf16")
    gc = oracle.num_groups(n, m)
    gmax = torch.full((1, h, gc, n), -1.0, device="cuda", dtype=torch.float32)
    ws = workspace(_lib.FGA_WS_CACHED_GROUP_MAX, _lib.shape(1, h, n, d, m))
    qd, kd = to_bf16_dev(q), to_bf16_dev(k)  # held: ptr() of a temporary would let k reuse q's block
    _lib.call("fga_cached_group_max", ptr(qd), ptr(kd), _lib.shape(1, h, n, d, m), 1, ptr(gmax), ptr(ws), ws.numel(),
              stream())
    torch.cuda.synchronize()
    got = gmax.cpu().numpy()
    mism = got != ref
    print(f"cached group max: {mism.mean():.2e} of values differ (n={n}, cc={cc})")
    assert mism.mean() < 1e-4  # measured <= 6.3e-5
    if mism.any():
        rel = np.abs(got[mism] - ref[mism]) / np.maximum(np.abs(ref[mism]), 1e-30)
        assert rel.max() <= 2 ** -7
    assert (((got >= 0.5 / n) != keep_ref) <= mism).all()


@pytest.mark.parametrize("n,distinct", [(5000, 7), (32760, 300), (40000, 3), (90000, 5)])
def test_topk_keep_many_ties(n, distinct):
    # rows whose k-th largest value is shared by hundreds to thousands of keys (the builders'
    # bf16-valued scores): exactly k kept, ties toward the smaller index (masks.py:144-145,
    # lexsort((arange, -s))); n = 90000 takes the long-row ordered pass
    rng = np.random.default_rng(n)
    rows = 6
    vals = rng.standard_normal(distinct).astype(np.float32)
    scores = vals[rng.integers(0, distinct, size=(rows, n))]
    keep = torch.empty((rows, n), dtype=torch.uint8, device="cuda")
    sd = torch.from_numpy(scores).cuda()
    for k in (1, n // 3, n // 2 + 7, n - 1):
        _lib.call("fga_topk_keep", ptr(sd), rows, n, k, ptr(keep), stream())
        torch.cuda.synchronize()
        got = keep.cpu().numpy()
        for r in range(rows):
            order = np.lexsort((np.arange(n), -scores[r]))[:k]
            ref = np.zeros(n, np.uint8)
            ref[order] = 1
            assert np.array_equal(got[r], ref), (n, k, r)
