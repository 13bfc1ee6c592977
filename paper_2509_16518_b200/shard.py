"""Multi-GPU sharding of the operator (one process per GPU, no hot-path collective).

Every (b, h, g) work unit reads only its own query rows, its own key list and
the K/V of head (b, h) (/root/reference/pkg/src/sliceattn/sparse.py:138-155),
so units are independent.  Two layouts:

* ``partition_tiles`` -- contiguous runs of head-major tiles balanced by the
  pair work ``rows_g * count_g`` (the roofline numerator).  Runs of tiles are
  (head, group-range) units, so e.g. 12 heads split evenly over 8 GPUs.
  Each rank launches ``sparse_attention_shard`` on its range.
* ``head_blocks`` -- contiguous head blocks (the 40-head Wan 14B case).

Outputs are assembled only for validation (``gather_outputs``, an NCCL
all-gather outside any timed region).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import ptr, stream_ptr, torch
from .core import AttnConfig
from .sparse import DeviceIndexMask, _as_device_mask

__all__ = ["tile_work", "partition_tiles", "head_blocks", "sparse_attention_shard", "gather_outputs"]


def tile_work(cfg: AttnConfig, counts) -> np.ndarray:
    """Pair work of every tile in launch order (head-major, 128-row sub-tiles)."""
    c = np.asarray(counts, dtype=np.int64).reshape(cfg.batch * cfg.heads, cfg.num_groups)
    tpg = -(-cfg.group_size // 128)
    rows = []
    for g in range(cfg.num_groups):
        lo, hi = cfg.group_bounds(g)
        rows.append([max(0, min(128, hi - lo - 128 * s)) for s in range(tpg)])
    rows = np.array(rows, dtype=np.int64)                      # [G, tpg]
    return (c[:, :, None] * rows[None, :, :]).reshape(-1)      # [B*H*G*tpg]


def partition_tiles(work: np.ndarray, parts: int) -> list[tuple[int, int]]:
    """Split [0, len(work)) into ``parts`` contiguous ranges of near-equal total work."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    n = len(work)
    cum = np.concatenate([[0], np.cumsum(work, dtype=np.int64)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, parts):
        cuts.append(int(np.searchsorted(cum, total * r / parts, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.minimum(np.array(cuts), n))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(parts)]


def head_blocks(heads: int, parts: int) -> list[tuple[int, int]]:
    """Contiguous head blocks, sizes differing by at most one."""
    base, extra = divmod(heads, parts)
    out, h0 = [], 0
    for r in range(parts):
        h1 = h0 + base + (1 if r < extra else 0)
        out.append((h0, h1))
        h0 = h1
    return out


def sparse_attention_shard(qd, kd, vd, mask: DeviceIndexMask, cfg: AttnConfig, tile_range, out):
    """Run tiles [begin, end) of the full problem into ``out`` (full-size CUDA tensor)."""
    t = torch()
    b, e = tile_range
    mask = _as_device_mask(mask, cfg, qd.device.index)
    _lib.call("fga_sparse_attn_fwd_tiles", ptr(qd), ptr(kd), ptr(vd), ptr(mask.idx), mask.stride, ptr(mask.counts),
              ptr(out), _lib.FGA_OUT_F32 if out.dtype == t.float32 else _lib.FGA_OUT_BF16, None,
              _lib.shape(*cfg.dims, cfg.group_size, cfg.scale), int(b), int(e), stream_ptr())
    return out


def gather_outputs(local, group=None):
    """All-gather equally shaped per-rank tensors (validation only; NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist

    t = torch()
    world = dist.get_world_size(group)
    local = local.contiguous()
    if dist.get_backend(group) == "nccl":
        out = t.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local, group=group)
        return out
    parts = [t.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local, group=group)
    return t.stack(parts)
