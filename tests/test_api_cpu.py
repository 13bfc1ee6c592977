"""CPU-side tests of the drop-in API: validation/exceptions mirror the reference,
host-side mask plumbing and accounting match the reference goldens, the C-ABI
library loads and exports every declared symbol, and the product path refuses
to run without a GPU (no CPU fallback)."""

import ctypes
import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_2509_16518_b200 as fga
from conftest import ROOT
from paper_2509_16518_b200 import _lib


# ---------------------------------------------------------------- the C ABI boundary

def header_symbols():
    text = open(os.path.join(ROOT, "include", "fgattn.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fga_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_library_reports_version_and_no_device_here():
    lib = _lib.load()
    assert lib.fga_version() >= 100
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert lib.fga_device_supported(0) == 0


def test_cabi_validation_without_gpu():
    lib = _lib.load()
    bad = _lib.shape(1, 1, 100, 64, 200)   # group_size > seq_len
    rc = lib.fga_sparse_attn_fwd(1, 1, 1, 1, 100, 1, 1, 0, None, bad, None)
    assert rc == _lib.FGA_EINVAL
    assert b"group_size" in lib.fga_last_error()
    rc = lib.fga_sparse_attn_fwd(None, 1, 1, 1, 100, 1, 1, 0, None, _lib.shape(1, 1, 100, 64, 64), None)
    assert rc == _lib.FGA_EINVAL
    with pytest.raises(fga.ShapeError):
        _lib.check(rc, "x")


def test_workspace_sizes_without_gpu():
    # the library never allocates: every scratch buffer is sized by fga_workspace_bytes (host-only)
    shp = _lib.shape(1, 12, 32760, 128, 128)
    g = 256
    pooled = _lib.workspace_bytes(_lib.FGA_WS_POOLED_SCORES, shp)
    assert pooled >= 12 * g * 128 * 4 + 3 * 12 * g * 128 * 2           # q-bar fp32 + its 3 bf16 parts
    assert _lib.workspace_bytes(_lib.FGA_WS_CACHED_GROUP_MAX, shp) >= 12 * 32760 * (4 + 8)
    cells = 12 * g * 32760
    assert _lib.workspace_bytes(_lib.FGA_WS_BUILD_AVGQ, shp, 1) >= pooled + 2 * cells   # bf16 scores
    assert _lib.workspace_bytes(_lib.FGA_WS_BUILD_AVGQ, shp, 0) >= pooled + 5 * cells   # fp32 + keep bytes
    assert _lib.workspace_bytes(_lib.FGA_WS_BUILD_CACHED, shp) >= 5 * cells
    # tiny rows: the fused threshold's keep bits + empty-row list + count (three 256-byte-aligned
    # pieces) must fit even where the bf16 score buffer would be smaller
    tiny = _lib.shape(1, 3, 1, 64, 1)
    assert _lib.workspace_bytes(_lib.FGA_WS_BUILD_AVGQ, tiny, 1) >= \
        _lib.workspace_bytes(_lib.FGA_WS_POOLED_SCORES, tiny) + 3 * 256
    assert _lib.load().fga_workspace_bytes(99, shp, 1) == _lib.FGA_EINVAL
    assert _lib.load().fga_workspace_bytes(1, _lib.shape(1, 1, 10, 64, 20), 1) == _lib.FGA_EINVAL


def test_builder_and_select_argument_checks_without_gpu():
    # the reference's ValueErrors (masks.py:100-101, :139-140) and shape checks, before any launch
    lib = _lib.load()
    shp = _lib.shape(1, 1, 256, 64, 128)
    args = lambda strategy, tau, k, stride=256: (1, 1, shp, strategy, tau, k, 1, 1, stride, 1, 0, None, 0, None)
    assert lib.fga_build_mask_avgq(*args(_lib.FGA_SELECT_THRESHOLD, 0.0, 1)) == _lib.FGA_EINVAL  # tau <= 0
    assert b"tau" in lib.fga_last_error()
    assert lib.fga_build_mask_avgq(*args(_lib.FGA_SELECT_TOPK, 0.0, 257)) == _lib.FGA_EINVAL     # top_k > N
    assert lib.fga_build_mask_avgq(*args(7, 1.0, 1)) == _lib.FGA_EINVAL                          # strategy
    assert lib.fga_build_mask_avgq(*args(_lib.FGA_SELECT_TOPK, 0.0, 5, stride=100)) == _lib.FGA_EINVAL
    assert lib.fga_build_mask_cached(1, 1, shp, -1.0, 1, 1, 256, 1, 0, None, 0, None) == _lib.FGA_EINVAL
    assert lib.fga_select_compact(1, 2, 100, _lib.FGA_SELECT_TOPK, 0.0, 0, 1, 100, 1, 0, None) == _lib.FGA_EINVAL
    big = _lib.FGA_SELECT_MAX_N + 1
    assert lib.fga_select_compact(1, 2, big, _lib.FGA_SELECT_TOPK, 0.0, 1, 1, big, 1, 0, None) == _lib.FGA_EUNSUPPORTED
    # workspace alignment is checked before any launch
    assert lib.fga_pooled_scores(1, 1, shp, 1, 1, 8, 1 << 20, None) == _lib.FGA_EINVAL
    assert b"aligned" in lib.fga_last_error()


def test_product_path_has_no_cpu_fallback():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    cfg = fga.AttnConfig(1, 1, 256, 64, precision="bf16")
    q = fga.new_tensor(cfg, "gaussian", seed=1)
    with pytest.raises(RuntimeError, match="no CPU fallback|CUDA"):
        fga.sparse_attention(q, q, q, fga.full_mask(cfg), cfg)


# ---------------------------------------------------------------- config / tensors (core.py)

@pytest.mark.parametrize("kw", [dict(batch=0), dict(heads=-1), dict(seq_len=0), dict(head_dim=1.5),
                                dict(group_size=300), dict(scale=-1.0), dict(precision="fp8")])
def test_config_validation(kw):
    base = dict(batch=1, heads=1, seq_len=256, head_dim=64)
    base.update(kw)
    with pytest.raises(ValueError):
        fga.AttnConfig(**base)


def test_config_defaults_and_groups():
    cfg = fga.AttnConfig(1, 2, 1000, 64)
    assert cfg.scale == pytest.approx(1 / 8)
    assert cfg.num_groups == 8
    assert cfg.group_bounds(7) == (896, 1000)
    assert cfg.dims == (1, 2, 1000, 64)


def test_tensor_errors():
    with pytest.raises(fga.ShapeError):
        fga.AttnTensor(np.zeros((2, 2)))
    with pytest.raises(fga.NumericError):
        fga.AttnTensor(np.full((1, 1, 1, 1), np.inf))
    t = fga.AttnTensor(np.ones((1, 1, 2, 2)))
    assert not t.data.flags.writeable and t.data.dtype == np.float32
    cfg = fga.AttnConfig(1, 1, 4, 2, group_size=2)
    with pytest.raises(fga.ShapeError):
        fga.new_tensor(cfg, "from_data", data=np.zeros(7))
    with pytest.raises(ValueError):
        fga.new_tensor(cfg, "uniform")


def test_new_tensor_and_bf16_match_oracle(golden):
    g = golden("c1_random30")
    cfg = fga.AttnConfig(*g.shape, precision="bf16")
    q = fga.new_tensor(cfg, "gaussian", seed=1)
    assert np.array_equal(q.data, g.q)
    assert np.array_equal(fga.round_bf16(g.q), oracle.bf16_round(g.q))


def test_attn_map_validation():
    with pytest.raises(fga.ShapeError):
        fga.AttnMap(np.zeros((1, 1, 2, 3)))
    with pytest.raises(ValueError):
        fga.AttnMap(np.full((1, 1, 2, 2), 0.9))


# ---------------------------------------------------------------- masks (sparse.py) on the host

def test_mask_validation_mirrors_reference():
    with pytest.raises(fga.ShapeError):
        fga.SparseIndexMask(1, 1, 10, 20, [[[]]])
    with pytest.raises(fga.ShapeError):
        fga.SparseIndexMask(1, 1, 10, 5, [[[[0]]]])          # 1 group given, 2 needed
    with pytest.raises(ValueError):
        fga.SparseIndexMask(1, 1, 10, 5, [[[[0], []]]])       # empty group
    with pytest.raises(ValueError):
        fga.SparseIndexMask(1, 1, 10, 5, [[[[0], [10]]]])     # out of range
    m = fga.SparseIndexMask(1, 1, 10, 5, [[[[3, 1, 3], [9]]]])
    assert m.keys_for(0, 0, 0).tolist() == [1, 3]             # sorted + deduplicated


def test_random_mask_matches_reference_stream(golden):
    g = golden("c1_random30")
    cfg = fga.AttnConfig(*g.shape, precision="bf16")
    m = fga.random_mask(cfg, 0.3, seed=0)
    ref = g.lists()
    assert all(np.array_equal(m.keys_for(0, h, gg), ref[h * cfg.num_groups + gg])
               for h in range(2) for gg in range(cfg.num_groups))
    assert fga.mask_density(m) == pytest.approx(float(g["density"]))
    with pytest.raises(ValueError):
        fga.random_mask(cfg, 0.0)


@pytest.mark.parametrize("name", ["ragged_n1000", "lens_ragged", "m64_n300"])
def test_export_import_padded_roundtrip(golden, name):
    g = golden(name)
    b, h, n, d = g.shape
    m = fga.import_padded(g["padded"].astype(np.int32), g.group_size)
    assert np.array_equal(fga.export_padded(m), g["padded"].astype(np.int32))
    with pytest.raises(fga.ShapeError):
        fga.import_padded(g["padded"][..., :-1], g.group_size + 1000)


def test_export_padded_known_answer_and_interior_sentinel():
    m = fga.SparseIndexMask(1, 1, 4, 4, [[[[0, 2]]]])
    assert fga.export_padded(m).tolist() == [[[[0, 2, -1, -1]]]]
    with pytest.raises(ValueError):
        fga.import_padded(np.array([[[[0, -1, 2, -1]]]]), 4)


def test_full_mask_and_jaccard():
    cfg = fga.AttnConfig(1, 2, 256, 64)
    full = fga.full_mask(cfg)
    assert fga.mask_density(full) == 1.0
    r = fga.random_mask(cfg, 0.5, seed=3)
    assert fga.mask_jaccard(full, r) == pytest.approx(fga.mask_density(r))
    assert fga.mask_jaccard(r, r) == 1.0


def test_sparse_attention_argument_errors():
    cfg = fga.AttnConfig(1, 1, 256, 64)
    q = fga.new_tensor(cfg, "gaussian", seed=1)
    other = fga.AttnConfig(1, 2, 256, 64)
    with pytest.raises(fga.ShapeError):
        fga.sparse_attention(q, q, fga.new_tensor(other), fga.full_mask(cfg), cfg)
    with pytest.raises(fga.ShapeError):
        fga.sparse_attention(q, q, q, fga.full_mask(other), cfg)
    with pytest.raises(ValueError):
        fga.sparse_attention(q, q, q, fga.full_mask(cfg), cfg, chunk_size=129)


def test_mask_builder_config_validation():
    with pytest.raises(ValueError):
        fga.MaskBuilderConfig("nope")
    with pytest.raises(ValueError):
        fga.MaskBuilderConfig("avg_query_threshold", tau=0)
    with pytest.raises(ValueError):
        fga.MaskBuilderConfig("avg_query_topk", top_k=0)
    st = fga.CachedMaskState(mask=None, built_at_iteration=0, refresh_interval=15)
    assert not fga.refresh_policy(st, 14) and fga.refresh_policy(st, 15)   # SPEC: PAPER 5.1 cadence


# ---------------------------------------------------------------- accounting (perfmodel.py)

@pytest.mark.parametrize("name", ["c1_random30", "lens_ragged", "m64_n300", "full_n384"])
def test_count_flops_matches_reference(golden, name):
    g = golden(name)
    cfg = fga.AttnConfig(*g.shape, group_size=g.group_size, precision="bf16")
    m = fga.import_padded(g["padded"].astype(np.int32), g.group_size)
    rep = fga.count_flops(cfg, m).as_dict()
    ref = json.loads(str(g["count_flops"]))
    for key in ("flops_scores", "flops_output", "flops_softmax", "bytes_qkv", "bytes_mask", "flops_total"):
        assert rep[key] == ref[key], key
    trace = fga.synthetic_trace(cfg, m)
    assert [e.keys for e in trace] == list(g["trace_keys"])
    assert fga.trace_flops(trace, cfg.head_dim)[0] == ref["flops_scores"]


def test_dense_flops_identity():
    cfg = fga.AttnConfig(1, 2, 300, 64, group_size=64)
    dense = fga.count_flops(cfg, None)
    full = fga.count_flops(cfg, fga.full_mask(cfg))
    assert dense.flops_total == full.flops_total
    assert dense.flops_scores == 2 * 64 * 2 * 300 * 300
    assert fga.flop_speedup(dense, full, True) == 1.0


# ---------------------------------------------------------------- multi-GPU host logic

def test_partition_tiles_balanced_and_contiguous():
    from paper_2509_16518_b200 import shard

    cfg = fga.AttnConfig(1, 12, 32760, 128)
    rng = np.random.default_rng(0)
    counts = rng.integers(1000, 20000, size=(1, 12, cfg.num_groups))
    work = shard.tile_work(cfg, counts)
    assert work.sum() == fga.perfmodel.pair_count(cfg, None) * 0 + int(
        (counts[0] * np.array([min(128, 32760 - g * 128) for g in range(cfg.num_groups)])).sum())
    for parts in (1, 2, 3, 8):
        ranges = shard.partition_tiles(work, parts)
        assert ranges[0][0] == 0 and ranges[-1][1] == len(work)
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        loads = [work[a:b].sum() for a, b in ranges]
        assert max(loads) - min(loads) <= work.max()
    assert shard.head_blocks(40, 8) == [(5 * i, 5 * i + 5) for i in range(8)]
    assert shard.head_blocks(12, 8)[0] == (0, 2)


def _gloo_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import oracle as orc
    from paper_2509_16518_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, h, n, d, m = 1, 3, 512, 64, 128
    cfg = fga.AttnConfig(b, h, n, d, group_size=m)
    q, k, v = (orc.bf16_round(orc.gaussian((b, h, n, d), s)) for s in (1, 2, 3))
    lists = orc.random_lists(b, h, n, m, 0.4, seed=5)
    counts = np.array([len(x) for x in lists]).reshape(b, h, -1)
    ranges = shard.partition_tiles(shard.tile_work(cfg, counts), world)
    t0, t1 = ranges[rank]
    out = np.zeros((b, h, n, d), np.float32)
    g_count = cfg.num_groups
    for tile in range(t0, t1):           # one tile per group here (M = 128)
        hh, gg = divmod(tile, g_count)
        lo, hi = cfg.group_bounds(gg)
        out[0, hh, lo:hi] = orc.sparse_attention_group(q[0, hh, lo:hi], k[0, hh], v[0, hh], lists[tile], cfg.scale)
    allo = shard.gather_outputs(torch.from_numpy(out))
    if rank == 0:
        full = allo.sum(0).numpy()        # ranges are disjoint: rows of other ranks are zero
        ref = orc.chunked_sparse_attention(q, k, v, lists, m, None, "full")
        np.save(result_path, np.array([np.abs(full - ref).max(), float(len(ranges))]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_units_gloo_world2(tmp_path):
    import torch.multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    res = str(tmp_path / "r.npy")
    mp.spawn(_gloo_worker, args=(2, port, res), nprocs=2, join=True)
    err, parts = np.load(res)
    assert parts == 2 and err < 1e-5


def test_bench_reference_arm_prints_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sliceattn")):
        # the install is git-ignored; without it the arm must still print a contract line
        assert line["impl"] == "reference" and "unavailable" in line
        pytest.skip("baseline/_ref not installed (python -m pip install --no-index --target baseline/_ref ...)")
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "cpu_baseline", "e2e"):
        assert key in line
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
