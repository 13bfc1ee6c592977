"""B200-native FG-Attn: fine-grained (M x 1 slice) sparse attention.

Drop-in for the operator API of the reference package ``sliceattn``
(arXiv 2509.16518): same names, signatures, defaults and exceptions, with the
work done by hand-written sm_100a kernels in ``libfgattn.so`` (see
include/fgattn.h).  There is no CPU fallback.

    from paper_2509_16518_b200 import AttnConfig, new_tensor, random_mask, sparse_attention
    cfg = AttnConfig(1, 2, 4096, 64, precision="bf16")
    q, k, v = (new_tensor(cfg, "gaussian", seed=s) for s in (1, 2, 3))
    out = sparse_attention(q, k, v, random_mask(cfg, 0.3, seed=0), cfg)
"""

from .core import (GATHER, PRECISIONS, STREAM, AttnConfig, AttnMap, AttnTensor, NumericError, ShapeError,
                   TileEvent, analysis_scores, ingest, make_rng, new_tensor, round_bf16)
from .masks import (STRATEGIES, CachedMaskState, MaskBuilderConfig, block_sparsity, block_sparsity_qk, build_mask,
                    build_mask_avg_query, build_mask_cached, build_mask_cached_qk, cached_group_max,
                    pooled_query_scores, refresh_policy, slice_sparsity, slice_sparsity_qk)
from .pipeline import pack_keep_bits, sparse_attention_host
from .perfmodel import CostReport, count_flops, flop_speedup, synthetic_trace, trace_flops
from .sparse import (DeviceIndexMask, PackedTile, SparseIndexMask, compact_keep, compact_keep_bits, export_padded, full_mask,
                     gather_rows, import_padded, mask_density, mask_jaccard, masked_dense_attention, random_mask,
                     random_mask_device, sparse_attention)
from .tiled import OnlineSoftmaxState, dense_attention, finalize, flash_attention, init_state, online_softmax_update
from . import io  # noqa: E402  (FGT1 / FGM1 formats)
from .stream import IterStreamConfig, generate_stream, run_cached_pipeline

__version__ = "0.1.0"
