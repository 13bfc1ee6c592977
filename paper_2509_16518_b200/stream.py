"""Denoising-iteration stream and the cached-mask pipeline (reference SPEC.md:428-472).

The reference declares ``sliceattn.stream`` but ships none; this restates the spec on the
device path, which is how the paper deploys FG-Attn (the mask is recalibrated
every 15 DiT iterations and reused in between):

* ``generate_stream(sc)`` -- AR(1) snapshots: snapshot 0 is N(0, 1); snapshot t+1 =
  rho * snapshot_t + sqrt(1 - rho^2) * fresh N(0, 1), elementwise, so the marginal variance
  stays 1 and the lag-1 correlation is rho.  Deterministic per seed
  (a seeded torch generator on the device; one stream of Q, K, V per snapshot).
* ``run_cached_pipeline(stream, builder, cfg)`` -- per iteration: rebuild the mask on the
  GPU when ``refresh_policy`` says so (masks.py:55-57), run the sparse kernel with the
  cached mask, and report the mask density, its Jaccard overlap with a freshly built mask
  and the max-abs error of the output against dense attention and against the fresh mask's
  output.  Every tensor stays in HBM; only the report scalars come back.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from ._device import torch
from .core import AttnConfig
from .masks import CachedMaskState, MaskBuilderConfig, build_mask, refresh_policy
from .sparse import DeviceIndexMask, sparse_attention
from .tiled import flash_attention

__all__ = ["IterStreamConfig", "generate_stream", "run_cached_pipeline", "device_jaccard"]


@dataclass(frozen=True)
class IterStreamConfig:
    """cfg, iterations T >= 1, correlation rho in [0, 1], seed."""

    cfg: AttnConfig
    iterations: int
    rho: float
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if not 0.0 <= self.rho <= 1.0:
            raise ValueError("rho must lie in [0, 1]")


def generate_stream(sc: IterStreamConfig, device=None):
    """Yield T (Q, K, V) bf16 CUDA snapshots of the AR(1) process (fp32 state, bf16 views)."""
    t = torch()
    dev = t.device("cuda", t.cuda.current_device()) if device is None else t.device(device)
    gen = t.Generator(device=dev).manual_seed(sc.seed)
    shape = sc.cfg.dims
    state = [t.randn(shape, device=dev, dtype=t.float32, generator=gen) for _ in range(3)]
    a, b = float(sc.rho), math.sqrt(max(0.0, 1.0 - float(sc.rho) ** 2))
    for it in range(sc.iterations):
        if it > 0:
            for x in state:
                x.mul_(a).add_(t.randn(shape, device=dev, dtype=t.float32, generator=gen), alpha=b)
        yield tuple(x.to(t.bfloat16) for x in state)


def device_jaccard(a: DeviceIndexMask, b: DeviceIndexMask) -> float:
    """|A ∩ B| / |A ∪ B| over all (b, h, g, key) pairs of two device masks (mask_jaccard,
    sparse.py:235-250, on the GPU through keep bits)."""
    t = torch()
    n = a.seq_len
    rows = a.batch * a.heads * a.num_groups

    def keep(m):
        col = t.arange(m.stride, device=m.idx.device, dtype=t.int32)
        live = (col < m.counts.reshape(-1, 1)).reshape(rows, m.stride)
        k = t.zeros((rows, n + 1), dtype=t.bool, device=m.idx.device)
        idx = t.where(live, m.idx.reshape(rows, m.stride).long(), t.full_like(live, n, dtype=t.long))
        k.scatter_(1, idx, True)
        return k[:, :n]

    ka, kb = keep(a), keep(b)
    inter = int((ka & kb).sum().item())
    union = int((ka | kb).sum().item())
    return inter / union if union else 1.0


def run_cached_pipeline(stream, builder: MaskBuilderConfig, cfg: AttnConfig):
    """Per-iteration report dicts: iteration, refreshed, density, jaccard_vs_fresh,
    max_err_vs_dense, max_err_vs_fresh."""
    t = torch()
    state = None
    reports = []
    for it, (q, k, v) in enumerate(stream):
        fresh = build_mask(q, k, cfg, builder, device_result=True)
        refreshed = state is None or refresh_policy(state, it)
        if refreshed:
            state = CachedMaskState(mask=fresh, built_at_iteration=it, refresh_interval=builder.refresh_interval)
        mask = state.mask
        out = sparse_attention(q, k, v, mask, cfg, out_dtype=t.float32)
        out_fresh = out if mask is fresh else sparse_attention(q, k, v, fresh, cfg, out_dtype=t.float32)
        dense = flash_attention(q, k, v, cfg, out_dtype=t.float32)   # dense_attention (oracle.py:29-42), fp32 out
        total = cfg.batch * cfg.heads * cfg.num_groups * cfg.seq_len
        reports.append({
            "iteration": it,
            "refreshed": bool(refreshed),
            "density": mask.total_indices / total,
            "jaccard_vs_fresh": 1.0 if mask is fresh else device_jaccard(mask, fresh),
            "max_err_vs_dense": float((out - dense).abs().max().item()),
            "max_err_vs_fresh": float((out - out_fresh).abs().max().item()),
        })
    return reports
