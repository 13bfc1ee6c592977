"""Dense attention on the same tcgen05 pipeline (the speed-up denominator).

Mirror of /root/reference/pkg/src/sliceattn/tiled.py:80-114 (flash_attention)
and oracle.py:29-42 (dense_attention): every group attends to all N keys,
streamed as contiguous 128-key TMA tiles (fga_dense_attn_fwd) instead of
gathered ones.  The reference's per-tile helpers (init_state /
online_softmax_update / finalize, tiled.py:27-77) are what the kernel's softmax
warps do per chunk; they are also exported here, same names and semantics, as
fp32 device (torch) functions for callers that fold tiles themselves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import as_device_bf16, is_torch, ptr, stream_ptr, torch
from ._device import require_device
from .core import STREAM, AttnConfig, AttnTensor, NumericError, ShapeError
from .sparse import _check_qkv

__all__ = ["flash_attention", "dense_attention", "OnlineSoftmaxState", "init_state", "online_softmax_update",
           "finalize"]


@dataclass(frozen=True, eq=False)
class OnlineSoftmaxState:
    """Running softmax over the key tiles seen so far (tiled.py:27-37): running_max [rows],
    denom [rows], acc [rows, head_dim], fp32 CUDA tensors."""

    running_max: object
    denom: object
    acc: object


def _dev_f32(x):
    t = torch()
    if is_torch(x):
        return x.to(t.float32)
    return t.as_tensor(np.asarray(x, dtype=np.float32), device=f"cuda:{require_device()}")


def init_state(rows: int, head_dim: int) -> OnlineSoftmaxState:
    """tiled.py:40-45."""
    t = torch()
    dev = f"cuda:{require_device()}"
    return OnlineSoftmaxState(running_max=t.full((rows,), -float("inf"), dtype=t.float32, device=dev),
                              denom=t.zeros(rows, dtype=t.float32, device=dev),
                              acc=t.zeros((rows, head_dim), dtype=t.float32, device=dev))


def online_softmax_update(state: OnlineSoftmaxState, scores, values) -> OnlineSoftmaxState:
    """Fold one [rows, tile] tile of raw scores and its [tile, head_dim] values (tiled.py:48-71),
    with the same -inf guard: while no finite score has been seen the shift is 0."""
    t = torch()
    s, v = _dev_f32(scores), _dev_f32(values)
    if s.ndim != 2 or s.shape[1] < 1:
        raise ShapeError("scores must be [rows, tile] with tile >= 1")
    if v.shape[0] != s.shape[1]:
        raise ShapeError("values rows must match score columns")
    new_max = t.maximum(state.running_max, s.max(dim=1).values)
    safe = t.where(t.isneginf(new_max), t.zeros_like(new_max), new_max)
    rescale = t.exp(state.running_max - safe)
    p = t.exp(s - safe[:, None])
    return OnlineSoftmaxState(running_max=new_max, denom=rescale * state.denom + p.sum(dim=1),
                              acc=rescale[:, None] * state.acc + p @ v)


def finalize(state: OnlineSoftmaxState):
    """acc / denom (tiled.py:74-77); NumericError on an empty denominator."""
    if not bool((state.denom > 0).all()):
        raise NumericError("online softmax finalized with an empty denominator")
    return state.acc / state.denom[:, None]


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
