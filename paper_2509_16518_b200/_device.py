"""Device plumbing: torch owns memory and streams; libfgattn.so does the work.

No CPU fallback: every entry point calls ``require_device()``, which raises
unless a CUDA device of compute capability 10.0 (sm_100) is present and the
in-tree ``libfgattn.so`` loads.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_checked: dict[int, bool] = {}


def torch():
    import torch as _t

    return _t


def require_device(device=None) -> int:
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2509_16518_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    dev = t.cuda.current_device() if device is None else t.device(device).index
    if dev is None:
        dev = t.cuda.current_device()
    if dev not in _checked:
        lib = _lib.load()
        if not lib.fga_device_supported(int(dev)):
            cap = t.cuda.get_device_capability(dev)
            raise RuntimeError(f"device {dev} has compute capability {cap}; libfgattn.so is built for sm_100a")
        _checked[dev] = True
    return dev


def stream_ptr():
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def is_torch(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor)


def host_array(x) -> np.ndarray:
    """fp32 host array of an AttnTensor / AttnMap / ndarray."""
    data = getattr(x, "data", x)
    return np.asarray(data, dtype=np.float32)


def as_device_bf16(x, device=None):
    """Contiguous bf16 CUDA tensor from a torch tensor or host fp32 data (RNE cast)."""
    t = torch()
    dev = require_device(device)
    if isinstance(x, t.Tensor):
        y = x
        if not y.is_cuda:
            y = y.to(f"cuda:{dev}")
        if y.dtype != t.bfloat16:
            y = y.to(t.bfloat16)
        return y.contiguous()
    arr = host_array(x)
    return t.from_numpy(np.ascontiguousarray(arr)).to(f"cuda:{dev}").to(t.bfloat16).contiguous()


def as_device(x, dtype, device=None):
    t = torch()
    dev = require_device(device)
    if isinstance(x, t.Tensor):
        return x.to(device=f"cuda:{dev}", dtype=dtype).contiguous()
    return t.as_tensor(np.ascontiguousarray(x)).to(device=f"cuda:{dev}", dtype=dtype).contiguous()
