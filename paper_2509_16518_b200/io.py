"""Bit-exact file formats for tensors, maps and slice masks (reference SPEC.md:474-511).

The reference declares an ``io`` module (pkg/pyproject.toml package list, SPEC.md [MODULE] io)
but ships none; this is a restatement of the specified formats, little-endian throughout:

* ``FGT1`` tensor / map: magic ``b"FGT1"``, version u16 (1), dtype code u16 (0 = f32), rank u32,
  dims u64 x rank, then the row-major payload.
* ``FGM1`` mask: magic ``b"FGM1"``, version u16 (1), reserved u16 (0), then B, H, G, N, M as u64,
  then for every (b, h, g) in flat order (b*H + h)*G + g a u32 length followed by that many sorted
  u32 key indices (the compact form of the paper's index array).

Errors follow the spec: a bad magic / version raises ``FormatError``, a payload that does not
match its header (truncated, trailing bytes, dimension overflow, bad list) raises
``CorruptionError``.  ``read_mask_device`` decodes straight into the device
index layout the kernels consume (the same ``[B, H, G, N]`` int32 + counts as ``compact_keep``).
"""

from __future__ import annotations

import struct

import numpy as np

from .core import AttnMap, AttnTensor
from .sparse import DeviceIndexMask, SparseIndexMask

_FGT1 = b"FGT1"
_FGM1 = b"FGM1"
_VERSION = 1
_DTYPES = {0: np.dtype("<f4")}


class FormatError(ValueError):
    """Unknown magic, version or dtype code."""


class CorruptionError(ValueError):
    """Payload inconsistent with its header (truncated, oversized, invalid lists)."""


# ------------------------------------------------------------------ tensors / maps (FGT1)

def encode_tensor(array) -> bytes:
    data = np.ascontiguousarray(getattr(array, "data", array), dtype="<f4")
    head = _FGT1 + struct.pack("<HHI", _VERSION, 0, data.ndim) + struct.pack(f"<{data.ndim}Q", *data.shape)
    return head + data.tobytes()


def decode_tensor(buf: bytes) -> np.ndarray:
    mv = memoryview(buf)
    if len(mv) < 12 or bytes(mv[:4]) != _FGT1:
        raise FormatError("not an FGT1 tensor (bad magic)")
    version, dcode, rank = struct.unpack_from("<HHI", mv, 4)
    if version != _VERSION:
        raise FormatError(f"unsupported FGT1 version {version}")
    if dcode not in _DTYPES:
        raise FormatError(f"unsupported FGT1 dtype code {dcode}")
    off = 12
    if len(mv) < off + 8 * rank:
        raise CorruptionError("truncated FGT1 header")
    dims = struct.unpack_from(f"<{rank}Q", mv, off)
    off += 8 * rank
    dt = _DTYPES[dcode]
    count = 1
    for d in dims:
        count *= d
        if count * dt.itemsize > len(mv):
            raise CorruptionError("FGT1 dimensions exceed the payload")
    if len(mv) - off != count * dt.itemsize:
        raise CorruptionError(f"FGT1 payload is {len(mv) - off} bytes, header says {count * dt.itemsize}")
    return np.frombuffer(mv[off:], dtype=dt).reshape(dims).astype(np.float32)


def write_tensor(path: str, tensor) -> None:
    with open(path, "wb") as f:
        f.write(encode_tensor(tensor))


def read_tensor(path: str) -> AttnTensor:
    with open(path, "rb") as f:
        return AttnTensor(decode_tensor(f.read()))


def write_map(path: str, map_) -> None:
    write_tensor(path, map_)


def read_map(path: str) -> AttnMap:
    with open(path, "rb") as f:
        return AttnMap(decode_tensor(f.read()))


# ------------------------------------------------------------------ slice masks (FGM1)

def _mask_lists(mask) -> tuple[tuple[int, int, int, int, int], list[np.ndarray]]:
    if isinstance(mask, DeviceIndexMask):
        mask = mask.to_host()
    b, h, n, m = mask.batch, mask.heads, mask.seq_len, mask.group_size
    g = -(-n // m)
    lists = [np.asarray(mask.keys_for(bb, hh, gg), dtype=np.int64)
             for bb in range(b) for hh in range(h) for gg in range(g)]
    return (b, h, g, n, m), lists


def encode_mask(mask) -> bytes:
    (b, h, g, n, m), lists = _mask_lists(mask)
    parts = [_FGM1, struct.pack("<HH5Q", _VERSION, 0, b, h, g, n, m)]
    for lst in lists:
        parts.append(struct.pack("<I", len(lst)))
        parts.append(lst.astype("<u4").tobytes())
    return b"".join(parts)


def _parse_mask(buf: bytes):
    mv = memoryview(buf)
    if len(mv) < 8 or bytes(mv[:4]) != _FGM1:
        raise FormatError("not an FGM1 mask (bad magic)")
    version, _ = struct.unpack_from("<HH", mv, 4)
    if version != _VERSION:
        raise FormatError(f"unsupported FGM1 version {version}")
    if len(mv) < 48:
        raise CorruptionError("truncated FGM1 header")
    b, h, g, n, m = struct.unpack_from("<5Q", mv, 8)
    if m < 1 or n < 1 or m > n or g != -(-n // m):
        raise CorruptionError(f"inconsistent FGM1 header (B={b}, H={h}, G={g}, N={n}, M={m})")
    words = np.frombuffer(mv[48:], dtype="<u4") if (len(mv) - 48) % 4 == 0 else None
    if words is None:
        raise CorruptionError("FGM1 payload is not a whole number of u32 words")
    rows = b * h * g
    if b < 1 or h < 1 or rows > len(words):  # every row needs at least its length word
        raise CorruptionError(f"FGM1 header dims (B={b}, H={h}, G={g}) overflow the {len(words)}-word payload")
    starts = np.empty(rows, np.int64)
    lens = np.empty(rows, np.int64)
    pos = 0
    for r in range(rows):                    # lengths are interleaved with the lists: a serial walk
        if pos >= len(words):
            raise CorruptionError("truncated FGM1 payload")
        ln = int(words[pos])
        starts[r], lens[r] = pos + 1, ln
        pos += 1 + ln
        if pos > len(words):
            raise CorruptionError("truncated FGM1 payload")
    if pos != len(words):
        raise CorruptionError("trailing bytes after the FGM1 payload")
    return (b, h, g, n, m), words, starts, lens


def _check_lists(words, starts, lens, n):
    for s, ln in zip(starts, lens):
        lst = words[s:s + ln]
        if ln == 0:
            raise CorruptionError("empty key list (every (b,h,g) needs at least one key)")
        if int(lst.max()) >= n or (ln > 1 and not np.all(lst[1:] > lst[:-1])):
            raise CorruptionError("FGM1 lists must be strictly ascending indices < N")


def decode_mask(buf: bytes) -> SparseIndexMask:
    (b, h, g, n, m), words, starts, lens = _parse_mask(buf)
    _check_lists(words, starts, lens, n)
    flat = []
    for s, ln in zip(starts, lens):
        a = words[s:s + ln].astype(np.int64)
        a.flags.writeable = False
        flat.append(a)
    return SparseIndexMask._from_flat(b, h, n, m, flat)


def write_mask(path: str, mask) -> None:
    with open(path, "wb") as f:
        f.write(encode_mask(mask))


def read_mask(path: str) -> SparseIndexMask:
    with open(path, "rb") as f:
        return decode_mask(f.read())


def read_mask_device(path_or_bytes, device=None, fill_sentinel: bool = False) -> DeviceIndexMask:
    """FGM1 -> device ``[B, H, G, N]`` int32 index layout + counts, without building Python
    lists: the payload is uploaded once and scattered on the GPU by ``fga_fgm1_unpack``."""
    import torch

    from . import _lib

    buf = path_or_bytes
    if isinstance(path_or_bytes, str):
        with open(path_or_bytes, "rb") as f:
            buf = f.read()
    (b, h, g, n, m), words, starts, lens = _parse_mask(buf)
    _check_lists(words, starts, lens, n)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    payload = torch.from_numpy(words.view(np.int32).copy()).to(dev)
    starts_d = torch.from_numpy(starts).to(dev)
    idx = torch.empty((b, h, g, n), dtype=torch.int32, device=dev)
    counts = torch.empty((b, h, g), dtype=torch.int32, device=dev)
    _lib.call("fga_fgm1_unpack", payload.data_ptr(), starts_d.data_ptr(), b * h * g, n, idx.data_ptr(), n,
              counts.data_ptr(), 1 if fill_sentinel else 0, torch.cuda.current_stream(dev).cuda_stream)
    # _check_lists enforced the SparseIndexMask invariants on the host
    return DeviceIndexMask(idx=idx, counts=counts, batch=b, heads=h, seq_len=n, group_size=m, validated=True)
