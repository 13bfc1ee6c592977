"""FLOP / byte accounting of the operator (the measurement definition).

Mirror of the counting half of /root/reference/pkg/src/sliceattn/perfmodel.py
(:21-143): per computed (query row, key) pair 2*D FLOPs for the scores, 2*D
for the output and SOFTMAX_FLOPS_PER_SCORE for the softmax.  bench.py's
roofline numerator is ``flops_scores + flops_output`` of ``count_flops``.
The reference's illustrative cycle model (perfmodel.py:146-224) is out of
scope: real CUDA-event timings and ncu counters replace it.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from .core import GATHER, STREAM, AttnConfig, TileEvent

__all__ = ["SOFTMAX_FLOPS_PER_SCORE", "INDEX_BYTES", "ELEMENT_BYTES", "CostReport", "pair_count", "count_flops",
           "synthetic_trace", "trace_flops", "flop_speedup"]

SOFTMAX_FLOPS_PER_SCORE = 4
INDEX_BYTES = 4
ELEMENT_BYTES = 4


@dataclass(frozen=True)
class CostReport:
    """Work and data-movement totals of one workload (perfmodel.py:47-67)."""

    flops_scores: int
    flops_output: int
    flops_softmax: int
    bytes_qkv: int
    bytes_mask: int
    density: float
    modeled_cycles: int = 0
    projected_speedup: float = 1.0

    @property
    def flops_total(self) -> int:
        return self.flops_scores + self.flops_output + self.flops_softmax

    @property
    def flops_matmul(self) -> int:
        return self.flops_scores + self.flops_output

    def as_dict(self) -> dict:
        d = asdict(self)
        d["flops_total"] = self.flops_total
        return d


def _counts(mask) -> np.ndarray:
    if hasattr(mask, "counts") and callable(mask.counts):
        return np.asarray(mask.counts())
    if hasattr(mask, "counts"):  # DeviceIndexMask
        return mask.counts.cpu().numpy()
    return np.array([[[mask.keys_for(b, h, g).size for g in range(mask.num_groups)]
                      for h in range(mask.heads)] for b in range(mask.batch)])


def _group_rows(cfg: AttnConfig) -> np.ndarray:
    return np.array([hi - lo for lo, hi in (cfg.group_bounds(g) for g in range(cfg.num_groups))], dtype=np.int64)


def pair_count(cfg: AttnConfig, mask=None) -> int:
    """sum over groups of rows_g * |list_g|; B*H*N^2 when dense (perfmodel.py:70-81)."""
    if mask is None:
        return cfg.batch * cfg.heads * cfg.seq_len * cfg.seq_len
    c = _counts(mask).reshape(cfg.batch, cfg.heads, cfg.num_groups).astype(np.int64)
    return int((c * _group_rows(cfg)[None, None, :]).sum())


def count_flops(cfg: AttnConfig, mask=None) -> CostReport:
    """Counts-only report (perfmodel.py:92-110)."""
    if mask is not None:
        mask.check_compatible(cfg)
    pairs = pair_count(cfg, mask)
    if mask is None:
        streamed = cfg.batch * cfg.heads * cfg.num_groups * cfg.seq_len
        density = 1.0
    else:
        streamed = int(_counts(mask).sum())
        density = streamed / (cfg.batch * cfg.heads * cfg.num_groups * cfg.seq_len)
    io_rows = cfg.batch * cfg.heads * cfg.seq_len
    return CostReport(
        flops_scores=2 * pairs * cfg.head_dim,
        flops_output=2 * pairs * cfg.head_dim,
        flops_softmax=SOFTMAX_FLOPS_PER_SCORE * pairs,
        bytes_qkv=ELEMENT_BYTES * cfg.head_dim * (2 * io_rows + 2 * streamed),
        bytes_mask=0 if mask is None else INDEX_BYTES * streamed,
        density=density,
    )


def synthetic_trace(cfg: AttnConfig, mask=None) -> list[TileEvent]:
    """Tile stream of the kernels (perfmodel.py:113-132): G*ceil(N/M) STREAM
    tiles per head when dense, ceil(|list|/M) GATHER tiles per group otherwise."""
    m = cfg.group_size
    out = []
    counts = None if mask is None else _counts(mask).reshape(cfg.batch, cfg.heads, cfg.num_groups)
    for b in range(cfg.batch):
        for h in range(cfg.heads):
            for g in range(cfg.num_groups):
                lo, hi = cfg.group_bounds(g)
                total, kind = (cfg.seq_len, STREAM) if counts is None else (int(counts[b, h, g]), GATHER)
                out.extend(TileEvent(b, h, g, hi - lo, min(m, total - s), kind) for s in range(0, total, m))
    return out


def trace_flops(trace, head_dim: int) -> tuple[int, int, int]:
    """(scores, output, softmax) FLOPs implied by a trace (perfmodel.py:135-143)."""
    pairs = sum(e.rows * e.keys for e in trace)
    return 2 * pairs * head_dim, 2 * pairs * head_dim, SOFTMAX_FLOPS_PER_SCORE * pairs


def flop_speedup(dense: CostReport, sparse: CostReport, include_softmax: bool) -> float:
    """Matmul-only or with-softmax FLOP ratio (perfmodel.py:197-203)."""
    if include_softmax:
        return dense.flops_total / sparse.flops_total
    return dense.flops_matmul / sparse.flops_matmul
