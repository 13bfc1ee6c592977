"""ctypes binding of libfgattn.so (include/fgattn.h).

The library is built in-tree by ``paper_2509_16518_b200._build``.  There is
no fallback: if the library is missing or the device is not an sm_100 part,
calls raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGA_LIB") or os.path.join(_HERE, "libfgattn.so")  # FGA_LIB: A/B builds

FGA_OK, FGA_EINVAL, FGA_ERANGE, FGA_ECUDA, FGA_EUNSUPPORTED = 0, -1, -2, -3, -4
FGA_OUT_BF16, FGA_OUT_F32 = 0, 1
FGA_STATUS_EMPTY, FGA_STATUS_RANGE, FGA_STATUS_STRIDE, FGA_STATUS_ORDER = 1, 2, 4, 8
FGA_ATTN_CHECK, FGA_ATTN_PER_TILE, FGA_ATTN_STATIC = 1, 2, 4
FGA_WS_POOLED_SCORES, FGA_WS_CACHED_GROUP_MAX, FGA_WS_BUILD_AVGQ, FGA_WS_BUILD_CACHED = 1, 2, 3, 4
FGA_SELECT_THRESHOLD, FGA_SELECT_TOPK = 0, 1
FGA_SELECT_MAX_N = 114688


class FgaShape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("heads", ctypes.c_int64), ("seq_len", ctypes.c_int64),
                ("head_dim", ctypes.c_int64), ("group_size", ctypes.c_int64), ("scale", ctypes.c_float)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_F = ctypes.c_float
_SZ = ctypes.c_size_t

_SIGS = {
    "fga_version": ([], _I),
    "fga_last_error": ([], ctypes.c_char_p),
    "fga_device_supported": ([_I], _I),
    "fga_compact": ([_P, _P, _I64, _I64, _P, _I64, _P, _I, _P], _I),
    "fga_pack_bits": ([_P, _I64, _I64, _P, _P], _I),
    "fga_compact_bits": ([_P, _I64, _I64, _P, _I64, _P, _I, _P], _I),
    "fga_fgm1_unpack": ([_P, _P, _I64, _I64, _P, _I64, _P, _I, _P], _I),
    "fga_sparse_attn_fwd": ([_P, _P, _P, _P, _I64, _P, _P, _I, _P, FgaShape, _P], _I),
    "fga_sparse_attn_fwd_tiles": ([_P, _P, _P, _P, _I64, _P, _P, _I, _P, FgaShape, _I64, _I64, _P], _I),
    "fga_sparse_attn_fwd_ex": ([_P, _P, _P, _P, _I64, _P, _P, _I, _P, FgaShape, _I64, _I64, _P, _P, _I, _P], _I),
    "fga_sparse_attn_fwd_timed": ([_P, _P, _P, _P, _I64, _P, _P, _I, _P, FgaShape, _I64, _I64, _P, _P, _I, _P, _I64,
                                   _P], _I),
    "fga_validate_mask": ([_P, _I64, _P, _I64, _I64, _P, _P], _I),
    "fga_tile_order": ([_P, FgaShape, _P, _P], _I),
    "fga_dense_attn_fwd": ([_P, _P, _P, _P, _I, _P, FgaShape, _P], _I),
    "fga_gather_rows": ([_P, _I64, _I64, _P, _I64, _P, _P], _I),
    "fga_gather_ring_probe": ([_P, _P, _I64, _I64, _P, _I64, _P, _P, _P, _P], _I),
    "fga_workspace_bytes": ([_I, FgaShape, _I], _I64),
    "fga_pooled_scores": ([_P, _P, FgaShape, _I, _P, _P, _SZ, _P], _I),
    "fga_pooled_scores_bf16": ([_P, _P, FgaShape, _P, _P, _SZ, _P], _I),
    "fga_select_compact": ([_P, _I64, _I64, _I, _F, _I64, _P, _I64, _P, _I, _P], _I),
    "fga_build_mask_avgq": ([_P, _P, FgaShape, _I, _F, _I64, _I, _P, _I64, _P, _I, _P, _SZ, _P], _I),
    "fga_build_mask_cached": ([_P, _P, FgaShape, _F, _I, _P, _I64, _P, _I, _P, _SZ, _P], _I),
    "fga_threshold_keep": ([_P, _I64, _F, _P, _P], _I),
    "fga_topk_keep": ([_P, _I64, _I64, _I64, _P, _P], _I),
    "fga_group_max_map": ([_P, _I64, _I64, _I64, _I, _P, _P], _I),
    "fga_cached_group_max": ([_P, _P, FgaShape, _I, _P, _P, _SZ, _P], _I),
    "fga_random_keep": ([_I64, _I64, _I64, ctypes.c_uint64, _P, _P], _I),
}
EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the C ABI; raise if the library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not found: build it with `python -m paper_2509_16518_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """Map a negative FGA_E* code to the reference exception classes."""
    if rc == FGA_OK:
        return
    msg = f"{what}: {load().fga_last_error().decode(errors='replace')}"
    if rc == FGA_EINVAL:
        raise ShapeError(msg)
    if rc == FGA_ERANGE:
        raise IndexError(msg)
    if rc == FGA_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def call_rc(name: str, *args) -> tuple[int, str]:
    """Raw return code and message, for callers that map codes themselves."""
    rc = getattr(load(), name)(*args)
    return rc, ("" if rc == FGA_OK else load().fga_last_error().decode(errors="replace"))


def workspace_bytes(op: int, shp: FgaShape, round_bf16: int = 1) -> int:
    """Device workspace an operation needs (the library never allocates)."""
    n = load().fga_workspace_bytes(int(op), shp, int(round_bf16))
    if n < 0:
        check(int(n), "fga_workspace_bytes")
    return int(n)


def shape(batch, heads, seq_len, head_dim, group_size, scale=None) -> FgaShape:
    return FgaShape(int(batch), int(heads), int(seq_len), int(head_dim), int(group_size),
                    float(scale) if scale is not None else 0.0)
