"""Dense attention on the same tcgen05 pipeline (the speed-up denominator).

Mirror of /root/reference/pkg/src/sliceattn/tiled.py:80-114 (flash_attention)
and oracle.py:29-42 (dense_attention): every group attends to all N keys,
streamed as contiguous 128-key TMA tiles (fga_dense_attn_fwd) instead of
gathered ones.  The reference's per-tile helpers (init_state /
online_softmax_update / finalize, tiled.py:27-77) are what the kernel's softmax
warps do per chunk; they are also exported here, same names, semantics and
(NumPy) types, computed on the device, for callers that fold tiles themselves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import as_device_bf16, is_torch, ptr, stream_ptr, torch
from ._device import require_device
from .core import STREAM, AttnConfig, AttnTensor, NumericError, ShapeError
from .sparse import _check_precision, _check_qkv

__all__ = ["flash_attention", "dense_attention", "OnlineSoftmaxState", "init_state", "online_softmax_update",
           "finalize"]


@dataclass(frozen=True, eq=False)
class OnlineSoftmaxState:
    """Running softmax over the key tiles seen so far (tiled.py:27-37): running_max [rows],
    denom [rows], acc [rows, head_dim], fp32.  NumPy arrays (the reference's types) or, from
    ``init_state(..., device=True)`` / torch inputs, CUDA tensors."""

    running_max: object
    denom: object
    acc: object


def _dev_f32(x):
    t = torch()
    if is_torch(x):
        return x.to(device=f"cuda:{require_device()}", dtype=t.float32)
    return t.as_tensor(np.asarray(x, dtype=np.float32), device=f"cuda:{require_device()}")


def _host_state(state: OnlineSoftmaxState) -> bool:
    return not is_torch(state.running_max)


def init_state(rows: int, head_dim: int, *, device: bool = False) -> OnlineSoftmaxState:
    """tiled.py:40-45: NumPy state like the reference, or CUDA tensors with ``device=True``."""
    if not device:
        return OnlineSoftmaxState(running_max=np.full(rows, -np.inf, dtype=np.float32),
                                  denom=np.zeros(rows, dtype=np.float32),
                                  acc=np.zeros((rows, head_dim), dtype=np.float32))
    t = torch()
    dev = f"cuda:{require_device()}"
    return OnlineSoftmaxState(running_max=t.full((rows,), -float("inf"), dtype=t.float32, device=dev),
                              denom=t.zeros(rows, dtype=t.float32, device=dev),
                              acc=t.zeros((rows, head_dim), dtype=t.float32, device=dev))


def online_softmax_update(state: OnlineSoftmaxState, scores, values) -> OnlineSoftmaxState:
    """Fold one [rows, tile] tile of raw scores and its [tile, head_dim] values (tiled.py:48-71),
    with the same -inf guard: while no finite score has been seen the shift is 0.  Computed on
    the device; a NumPy state comes back as NumPy (the reference's types), a device state stays."""
    t = torch()
    if np.ndim(scores) != 2 or np.shape(scores)[1] < 1:
        raise ShapeError("scores must be [rows, tile] with tile >= 1")
    if np.shape(values)[0] != np.shape(scores)[1]:
        raise ShapeError("values rows must match score columns")
    s, v = _dev_f32(scores), _dev_f32(values)
    m0, d0, a0 = (_dev_f32(x) for x in (state.running_max, state.denom, state.acc))
    new_max = t.maximum(m0, s.max(dim=1).values)
    safe = t.where(t.isneginf(new_max), t.zeros_like(new_max), new_max)
    rescale = t.exp(m0 - safe)
    p = t.exp(s - safe[:, None])
    out = (new_max, rescale * d0 + p.sum(dim=1), rescale[:, None] * a0 + p @ v)
    if _host_state(state):
        out = tuple(x.cpu().numpy() for x in out)
    return OnlineSoftmaxState(running_max=out[0], denom=out[1], acc=out[2])


def finalize(state: OnlineSoftmaxState):
    """acc / denom (tiled.py:74-77); NumericError on an empty denominator."""
    denom, acc = _dev_f32(state.denom), _dev_f32(state.acc)
    if not bool((denom > 0).all()):
        raise NumericError("online softmax finalized with an empty denominator")
    out = acc / denom[:, None]
    return out.cpu().numpy() if _host_state(state) else out


def flash_attention(q, k, v, cfg: AttnConfig, trace: list | None = None, *, out_dtype=None):
    """Dense attention via key tiling; host inputs -> fp32 AttnTensor, CUDA inputs -> CUDA tensor."""
    _check_qkv(cfg, q, k, v)
    _check_precision(cfg, q, k, v)
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
