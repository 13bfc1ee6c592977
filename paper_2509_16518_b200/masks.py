"""Training-free slice-mask construction on the GPU (K1a -> K1b).

Mirror of /root/reference/pkg/src/sliceattn/masks.py:21-150.  Builders:

  build_mask_cached(map_, cfg, tau)     masks.py:94-105   group max of an explicit map
  build_mask_cached_qk(q, k, cfg, tau)  same mask without materialising the [B,H,N,N] map
  pooled_query_scores(q, k, cfg)        masks.py:108-118
  build_mask_avg_query(q, k, cfg, b)    masks.py:121-150  (threshold / top-k)

Each ends in K1b compaction (fga_compact) with the argmax fallback, so the
key lists are the reference's ``_lists_from_keep`` (masks.py:75-91) for the
same keep bits.  Host inputs give a host ``SparseIndexMask``; CUDA inputs (or
``device_result=True``) give a ``DeviceIndexMask`` that never leaves HBM.

Scores are fp32 dot products of the bf16 operands (precision='bf16'
semantics, bf16-rounded before thresholding as analysis_scores does).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import as_device, as_device_bf16, is_torch, ptr, stream_ptr, torch
from .core import AttnConfig, ShapeError
from .sparse import DeviceIndexMask, compact_keep

__all__ = [
    "STRATEGIES", "MaskBuilderConfig", "CachedMaskState", "refresh_policy", "build_mask_cached",
    "build_mask_cached_qk", "pooled_query_scores", "build_mask_avg_query", "build_mask", "cached_group_max",
    "block_sparsity", "slice_sparsity", "block_sparsity_qk", "slice_sparsity_qk",
]

STRATEGIES = ("cached_threshold", "avg_query_threshold", "avg_query_topk")


@dataclass(frozen=True)
class MaskBuilderConfig:
    """Strategy + parameters (masks.py:21-43)."""

    strategy: str
    tau: float = 0.0
    top_k: int = 1
    refresh_interval: int = 15

    def __post_init__(self):
        if self.strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}")
        if self.strategy.endswith("threshold") and self.tau <= 0:
            raise ValueError("threshold strategies need tau > 0")
        if self.strategy == "avg_query_topk" and self.top_k < 1:
            raise ValueError("top_k must be >= 1")
        if self.refresh_interval < 1:
            raise ValueError("refresh_interval must be >= 1")


@dataclass(frozen=True)
class CachedMaskState:
    """A mask plus the iteration it was calibrated at (masks.py:46-52)."""

    mask: object
    built_at_iteration: int
    refresh_interval: int


def refresh_policy(state: CachedMaskState, iteration: int) -> bool:
    """True when the cached mask is due for recomputation (masks.py:55-57)."""
    return (iteration - state.built_at_iteration) >= state.refresh_interval


def _round(cfg: AttnConfig) -> int:
    return 1 if cfg.precision == "bf16" else 0


def _finish(keep, scores, cfg: AttnConfig, host: bool, nonempty: bool = False):
    """K1b compaction; with scores every list is non-empty (argmax fallback), and top-k keeps
    k >= 1 keys, so those masks are valid by construction (no device check before first use)."""
    dm = compact_keep(keep, cfg.group_size, scores)
    dm.validated = dm.validated or nonempty
    return dm.to_host() if host else dm


def _check_qk(cfg, q, k):
    for t_ in (q, k):
        dims = tuple(t_.shape) if is_torch(t_) else tuple(np.shape(getattr(t_, "data", t_)))
        if dims != cfg.dims:
            raise ShapeError(f"tensor dims {dims} do not match config {cfg.dims}")


def _shape(cfg: AttnConfig):
    return _lib.shape(*cfg.dims, cfg.group_size, cfg.scale)


def _workspace(op: int, cfg: AttnConfig, device):
    """Caller-owned device workspace for ``op`` (the C ABI never allocates): a uint8 tensor
    from torch's caching allocator (512-byte aligned)."""
    t = torch()
    n = _lib.workspace_bytes(op, _shape(cfg), _round(cfg))
    return t.empty(max(n, 1), dtype=t.uint8, device=device)


def pooled_query_scores(q, k, cfg: AttnConfig):
    """exp((k_j . mean_{i in g} q_i) * scale) / D as fp32 [B, H, G, N] (fga_pooled_scores)."""
    _check_qk(cfg, q, k)
    t = torch()
    host = not is_torch(q)
    qd, kd = as_device_bf16(q), as_device_bf16(k)
    s = t.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=t.float32, device=qd.device)
    ws = _workspace(_lib.FGA_WS_POOLED_SCORES, cfg, qd.device)
    _lib.call("fga_pooled_scores", ptr(qd), ptr(kd), _shape(cfg), _round(cfg), ptr(s), ptr(ws), ws.numel(),
              stream_ptr())
    return s.cpu().numpy() if host else s


def _threshold(scores, tau: float):
    t = torch()
    keep = t.empty(scores.shape, dtype=t.uint8, device=scores.device)
    _lib.call("fga_threshold_keep", ptr(scores), scores.numel(), float(tau), ptr(keep), stream_ptr())
    return keep


def _lists(cfg: AttnConfig, device):
    t = torch()
    idx = t.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=t.int32, device=device)
    cnt = t.empty((cfg.batch, cfg.heads, cfg.num_groups), dtype=t.int32, device=device)
    return idx, cnt


def build_mask_avg_query(q, k, cfg: AttnConfig, builder: MaskBuilderConfig, device_result: bool = False):
    """Avg-query builder (masks.py:121-150): threshold keeps s >= tau (argmax
    fallback); top-k keeps the top_k largest, ties toward the smaller index.

    One C call (fga_build_mask_avgq): pooled scores on the tensor cores written as bf16,
    then selection fused with the compaction (fga_select_compact); the [B,H,G,N] scores
    never exist in fp32 and no keep bytes are written.  Every list is non-empty, ascending
    and in range by construction."""
    _check_qk(cfg, q, k)
    if builder.strategy == "avg_query_threshold":
        strategy = _lib.FGA_SELECT_THRESHOLD
    elif builder.strategy == "avg_query_topk":
        strategy = _lib.FGA_SELECT_TOPK
        if builder.top_k > cfg.seq_len:
            raise ValueError(f"top_k {builder.top_k} exceeds seq_len {cfg.seq_len}")
    else:
        raise ValueError(f"strategy {builder.strategy!r} does not pool queries")
    host = not is_torch(q) and not device_result
    qd, kd = as_device_bf16(q), as_device_bf16(k)
    idx, cnt = _lists(cfg, qd.device)
    ws = _workspace(_lib.FGA_WS_BUILD_AVGQ, cfg, qd.device)
    _lib.call("fga_build_mask_avgq", ptr(qd), ptr(kd), _shape(cfg), strategy, float(builder.tau),
              int(builder.top_k), _round(cfg), ptr(idx), cfg.seq_len, ptr(cnt), 0, ptr(ws), ws.numel(), stream_ptr())
    dm = DeviceIndexMask(cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size, idx, cnt, validated=True)
    return dm.to_host() if host else dm


def build_mask_cached(map_, cfg: AttnConfig, tau: float, device_result: bool = False):
    """Cached-threshold builder from an explicit post-softmax map (masks.py:94-105):
    keep key j of group g iff max_{i in g} a_ij >= tau (argmax fallback)."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    t = torch()
    host = not is_torch(map_) and not device_result
    m = as_device(getattr(map_, "data", map_), t.float32)
    expected = (cfg.batch, cfg.heads, cfg.seq_len, cfg.seq_len)
    if tuple(m.shape) != expected:
        raise ShapeError(f"map dims {tuple(m.shape)} do not match config {expected}")
    gmax = t.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=t.float32, device=m.device)
    _lib.call("fga_group_max_map", ptr(m), cfg.batch * cfg.heads, cfg.seq_len, cfg.group_size, _round(cfg),
              ptr(gmax), stream_ptr())
    return _finish(_threshold(gmax, tau), gmax, cfg, host)


def cached_group_max(q, k, cfg: AttnConfig):
    """max_{i in g} softmax(q_i K^T * scale)_j as fp32 [B, H, G, N], computed from
    Q and K in three streaming passes (row max, row denominator, group max)."""
    _check_qk(cfg, q, k)
    t = torch()
    qd, kd = as_device_bf16(q), as_device_bf16(k)
    gmax = t.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=t.float32, device=qd.device)
    ws = _workspace(_lib.FGA_WS_CACHED_GROUP_MAX, cfg, qd.device)
    _lib.call("fga_cached_group_max", ptr(qd), ptr(kd), _shape(cfg), _round(cfg), ptr(gmax), ptr(ws), ws.numel(),
              stream_ptr())
    return gmax


def build_mask_cached_qk(q, k, cfg: AttnConfig, tau: float, device_result: bool = False):
    """The cached-threshold mask of ``build_mask_cached(attention_map(q, k))``
    without materialising the N x N map (B200 path for Wan-scale N): one C call,
    fga_build_mask_cached."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    _check_qk(cfg, q, k)
    host = not is_torch(q) and not device_result
    qd, kd = as_device_bf16(q), as_device_bf16(k)
    idx, cnt = _lists(cfg, qd.device)
    ws = _workspace(_lib.FGA_WS_BUILD_CACHED, cfg, qd.device)
    _lib.call("fga_build_mask_cached", ptr(qd), ptr(kd), _shape(cfg), float(tau), _round(cfg), ptr(idx),
              cfg.seq_len, ptr(cnt), 0, ptr(ws), ws.numel(), stream_ptr())
    dm = DeviceIndexMask(cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size, idx, cnt, validated=True)
    return dm.to_host() if host else dm


def build_mask(q, k, cfg: AttnConfig, builder: MaskBuilderConfig, device_result: bool = False):
    """Dispatch a MaskBuilderConfig ("slice mask or threshold" form of the operator)."""
    if builder.strategy == "cached_threshold":
        return build_mask_cached_qk(q, k, cfg, builder.tau, device_result)
    return build_mask_avg_query(q, k, cfg, builder, device_result)


# ------------------------------------------------------------------ sparsity analyzers (masks.py:153-184)
# Table-2 style statistics on the GPU.  The map forms take an explicit [B,H,N,N] map like
# the reference; the ``_qk`` forms compute the same numbers from Q and K with the fused
# group-max kernel (fga_cached_group_max), so Wan-scale N -- where the N x N map cannot be
# materialised on a CPU -- is analysable.

def _map_group_max(map_, group: int, rnd: int):
    t = torch()
    m = as_device(getattr(map_, "data", map_), t.float32)
    if m.dim() != 4 or m.shape[2] != m.shape[3]:
        raise ShapeError(f"expected [B, H, N, N] map, got {tuple(m.shape)}")
    b, h, n, _ = m.shape
    g = -(-n // group)
    gmax = t.empty((b, h, g, n), dtype=t.float32, device=m.device)
    _lib.call("fga_group_max_map", ptr(m), b * h, n, group, rnd, ptr(gmax), stream_ptr())
    return gmax


def _tile_fraction(gmax, block: int, tau: float) -> float:
    """Fraction of block x block tiles (rows already reduced to row-blocks in gmax) whose
    max is below tau, averaged over (b, h); a partial edge tile counts over its real extent."""
    t = torch()
    b, h, g, n = gmax.shape
    pad = (-n) % block
    gm = t.nn.functional.pad(gmax, (0, pad), value=-1.0) if pad else gmax   # -1 < tau: ignored by max
    tile_max = gm.reshape(b, h, g, -1, block).amax(dim=-1)
    return float((tile_max < tau).float().mean(dim=(2, 3)).mean().item())


def block_sparsity(map_, block: int, tau: float) -> float:
    """Fraction of block x block score tiles with every entry below tau (masks.py:153-173)."""
    n = int((getattr(map_, "data", map_)).shape[2])
    if not 1 <= block <= n:
        raise ValueError(f"block must be in [1, {n}]")
    return _tile_fraction(_map_group_max(map_, block, 0), block, tau)


def slice_sparsity(map_, cfg: AttnConfig, tau: float) -> float:
    """Fraction of (group, key) M x 1 slices whose scores all fall below tau (masks.py:176-184)."""
    dims = tuple((getattr(map_, "data", map_)).shape)
    if dims != (cfg.batch, cfg.heads, cfg.seq_len, cfg.seq_len):
        raise ShapeError(f"map dims {dims} do not match config")
    gmax = _map_group_max(map_, cfg.group_size, _round(cfg))
    return float((gmax < tau).float().mean().item())


def block_sparsity_qk(q, k, cfg: AttnConfig, block: int, tau: float) -> float:
    """block_sparsity(attention_map(q, k)) without the N x N map."""
    if not 1 <= block <= cfg.seq_len:
        raise ValueError(f"block must be in [1, {cfg.seq_len}]")
    bcfg = AttnConfig(cfg.batch, cfg.heads, cfg.seq_len, cfg.head_dim, group_size=block, scale=cfg.scale,
                      precision="full")
    return _tile_fraction(cached_group_max(q, k, bcfg), block, tau)


def slice_sparsity_qk(q, k, cfg: AttnConfig, tau: float) -> float:
    """slice_sparsity(attention_map(q, k), cfg, tau) without the N x N map."""
    return float((cached_group_max(q, k, cfg) < tau).float().mean().item())
