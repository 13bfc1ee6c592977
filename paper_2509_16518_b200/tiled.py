"""Dense attention on the same tcgen05 pipeline (the speed-up denominator).

Mirror of /root/reference/pkg/src/sliceattn/tiled.py:80-114 (flash_attention)
and oracle.py:29-42 (dense_attention): every group attends to all N keys,
streamed as contiguous 128-key TMA tiles (fga_dense_attn_fwd) instead of
gathered ones.  The reference's per-tile numpy helpers (init_state /
online_softmax_update / finalize) live inside the kernel's softmax warps.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import as_device_bf16, is_torch, ptr, stream_ptr, torch
from .core import STREAM, AttnConfig, AttnTensor, NumericError
from .sparse import _check_qkv

__all__ = ["flash_attention", "dense_attention"]


def flash_attention(q, k, v, cfg: AttnConfig, trace: list | None = None, *, out_dtype=None):
    """Dense attention via key tiling; host inputs -> fp32 AttnTensor, CUDA inputs -> CUDA tensor."""
    _check_qkv(cfg, q, k, v)
    t = torch()
    host = not is_torch(q)
    qd, kd, vd = as_device_bf16(q), as_device_bf16(k), as_device_bf16(v)
    dt = t.float32 if host else (out_dtype or t.bfloat16)
    o = t.empty(cfg.dims, dtype=dt, device=qd.device)
    _lib.call("fga_dense_attn_fwd", ptr(qd), ptr(kd), ptr(vd), ptr(o),
              _lib.FGA_OUT_F32 if dt == t.float32 else _lib.FGA_OUT_BF16, None,
              _lib.shape(*cfg.dims, cfg.group_size, cfg.scale), stream_ptr())
    if trace is not None:
        from .perfmodel import synthetic_trace

        trace.extend(e for e in synthetic_trace(cfg, None) if e.kind == STREAM)
    if host:
        out = o.cpu().numpy()
        if not np.isfinite(out).all():
            raise NumericError("non-finite attention output")
        return AttnTensor(out)
    return o


def dense_attention(q, k, v, cfg: AttnConfig):
    """softmax(Q K^T * scale) V (oracle.py:29-42) -- the dense kernel."""
    return flash_attention(q, k, v, cfg)
