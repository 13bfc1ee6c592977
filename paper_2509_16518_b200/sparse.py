"""FG-Attn sparse attention: masks, the gather primitive and the operator.

Drop-in mirror of /root/reference/pkg/src/sliceattn/sparse.py.  The numeric
work runs in libfgattn.so:

  sparse_attention  -> fga_sparse_attn_fwd   (K2 cp.async/gather4 producer + K3 tcgen05)
  gather_rows       -> fga_gather_rows       (K2 TMA gather4, bitwise)
  compact_keep      -> fga_compact           (K1b ballot/prefix-sum compaction)
  random_mask_device-> fga_random_keep + fga_compact

Two mask representations:
  * ``SparseIndexMask`` -- the reference's host type (sorted, deduplicated,
    non-empty int64 lists; sparse.py:20-84).  Converted once to the device
    layout and cached.
  * ``DeviceIndexMask`` -- the paper's index array in HBM:
    int32 ``idx[B, H, G, stride]`` (ascending prefix per group) plus
    ``counts[B, H, G]``; what K1b produces and K2/K3 consume.

Host inputs (AttnTensor / ndarray) give host outputs (AttnTensor, fp32);
torch CUDA bf16 inputs give device outputs.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._device import as_device, as_device_bf16, is_torch, ptr, require_device, stream_ptr, torch
from .core import GATHER, AttnConfig, AttnTensor, NumericError, ShapeError, TileEvent

__all__ = [
    "SparseIndexMask", "DeviceIndexMask", "PackedTile", "gather_rows", "sparse_attention",
    "masked_dense_attention", "mask_density", "export_padded", "import_padded", "full_mask", "random_mask",
    "random_mask_device", "compact_keep", "compact_keep_bits", "mask_jaccard", "chunk_trace",
]


# ---------------------------------------------------------------- host mask

class SparseIndexMask:
    """Per-(b, h, g) sorted unique non-empty key lists (sparse.py:20-84)."""

    def __init__(self, batch: int, heads: int, seq_len: int, group_size: int, lists):
        if group_size < 1 or group_size > seq_len:
            raise ShapeError(f"group_size {group_size} invalid for seq_len {seq_len}")
        self.batch, self.heads, self.seq_len, self.group_size = batch, heads, seq_len, group_size
        g = self.num_groups
        if len(lists) != batch or any(len(hl) != heads for hl in lists):
            raise ShapeError("mask nesting must be [batch][heads][groups]")
        flat = []
        for per_b in lists:
            for per_h in per_b:
                if len(per_h) != g:
                    raise ShapeError(f"expected {g} groups per head, got {len(per_h)}")
                for keys in per_h:
                    a = np.unique(np.asarray(keys, dtype=np.int64))
                    if a.size == 0:
                        raise ValueError("every group needs at least one key")
                    if a[0] < 0 or a[-1] >= seq_len:
                        raise ValueError(f"key index out of range [0, {seq_len})")
                    a.flags.writeable = False
                    flat.append(a)
        self._lists = tuple(flat)
        self._device = {}

    @classmethod
    def _from_flat(cls, batch, heads, seq_len, group_size, flat):
        m = cls.__new__(cls)
        m.batch, m.heads, m.seq_len, m.group_size = batch, heads, seq_len, group_size
        m._lists = tuple(flat)
        m._device = {}
        return m

    @property
    def num_groups(self) -> int:
        return -(-self.seq_len // self.group_size)

    @property
    def total_indices(self) -> int:
        return sum(a.size for a in self._lists)

    def keys_for(self, b: int, h: int, g: int) -> np.ndarray:
        return self._lists[(b * self.heads + h) * self.num_groups + g]

    def counts(self) -> np.ndarray:
        return np.array([a.size for a in self._lists], dtype=np.int64).reshape(
            self.batch, self.heads, self.num_groups)

    def check_compatible(self, cfg: AttnConfig) -> None:
        ours = (self.batch, self.heads, self.seq_len, self.group_size)
        theirs = (cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size)
        if ours != theirs:
            raise ShapeError(f"mask built for {ours}, config is {theirs}")

    def to_device(self, device=None) -> "DeviceIndexMask":
        """Upload once per device (cached): padded int32 rows, ascending prefix then -1.
        The lists were validated on construction, so the device mask is marked validated."""
        dev = require_device(device)
        if dev not in self._device:
            pad = _padded_host(self)
            t = torch()
            idx = t.from_numpy(pad).to(f"cuda:{dev}")
            cnt = t.from_numpy(self.counts().astype(np.int32)).to(f"cuda:{dev}")
            self._device[dev] = DeviceIndexMask(self.batch, self.heads, self.seq_len, self.group_size, idx, cnt,
                                                validated=True)
        return self._device[dev]

    def __eq__(self, other):
        if not isinstance(other, SparseIndexMask):
            return NotImplemented
        return ((self.batch, self.heads, self.seq_len, self.group_size)
                == (other.batch, other.heads, other.seq_len, other.group_size)
                and all(np.array_equal(a, b) for a, b in zip(self._lists, other._lists)))

    def __hash__(self):
        return hash((self.batch, self.heads, self.seq_len, self.group_size))


def _padded_host(mask: SparseIndexMask) -> np.ndarray:
    rows = len(mask._lists)
    n = mask.seq_len
    counts = np.fromiter((a.size for a in mask._lists), dtype=np.int64, count=rows)
    pad = np.full((rows, n), -1, dtype=np.int32)
    if rows:
        flat = np.concatenate(mask._lists).astype(np.int32)
        row_of = np.repeat(np.arange(rows), counts)
        col_of = np.arange(flat.size) - np.repeat(np.cumsum(counts) - counts, counts)
        pad[row_of, col_of] = flat
    return pad.reshape(mask.batch, mask.heads, mask.num_groups, n)


# ---------------------------------------------------------------- device mask

@dataclass(eq=False)
class DeviceIndexMask:
    """Device-resident index mask: ``idx[B,H,G,stride]`` int32 + ``counts[B,H,G]`` int32.

    ``idx[b,h,g,:counts[b,h,g]]`` lists the kept keys of group g, ascending; entries
    beyond the count are ignored by the kernels (they hold -1 when produced
    with ``fill_sentinel``).  This is the paper's [B, H, N/M, N] array
     and the output of K1b.

    ``validated`` records that the SparseIndexMask invariants (sparse.py:36-52:
    1 <= count, keys in [0, N), sorted and unique) hold; producers that guarantee
    them set it, anything else is checked once on the device (``validate``)
    before its first use.  Treat the tensors as immutable after that."""

    batch: int
    heads: int
    seq_len: int
    group_size: int
    idx: object
    counts: object
    validated: bool = False
    _order: object = field(default=None, repr=False)
    _full: object = field(default=None, repr=False)

    @property
    def num_groups(self) -> int:
        return -(-self.seq_len // self.group_size)

    @property
    def stride(self) -> int:
        return int(self.idx.shape[-1])

    @property
    def total_indices(self) -> int:
        return int(self.counts.sum(dtype=torch().int64).item())

    def check_compatible(self, cfg: AttnConfig) -> None:
        ours = (self.batch, self.heads, self.seq_len, self.group_size)
        theirs = (cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size)
        if ours != theirs:
            raise ShapeError(f"mask built for {ours}, config is {theirs}")

    def keys_for(self, b: int, h: int, g: int) -> np.ndarray:
        c = int(self.counts[b, h, g].item())
        return self.idx[b, h, g, :c].cpu().numpy().astype(np.int64)

    def check_layout(self, device=None) -> None:
        """The tensor contract of the kernels: int32, contiguous, [B,H,G,stride] / [B,H,G],
        on ``device``.  ShapeError otherwise (no device work)."""
        t = torch()
        want = (self.batch, self.heads, self.num_groups)
        for name, x in (("idx", self.idx), ("counts", self.counts)):
            if not is_torch(x) or not x.is_cuda:
                raise ShapeError(f"DeviceIndexMask.{name} must be a CUDA tensor")
            if x.dtype != t.int32:
                raise ShapeError(f"DeviceIndexMask.{name} must be int32, got {x.dtype}")
            if not x.is_contiguous():
                raise ShapeError(f"DeviceIndexMask.{name} must be contiguous")
            if device is not None and x.device.index != device:
                raise ShapeError(f"DeviceIndexMask.{name} is on cuda:{x.device.index}, the inputs on cuda:{device}")
        if tuple(self.idx.shape[:3]) != want or self.idx.dim() != 4 or self.stride < 1:
            raise ShapeError(f"idx must be [B, H, G, stride] with [B, H, G] = {want}, got {tuple(self.idx.shape)}")
        if tuple(self.counts.shape) != want:
            raise ShapeError(f"counts must be {want}, got {tuple(self.counts.shape)}")

    def validate(self) -> "DeviceIndexMask":
        """Raise like SparseIndexMask would (sparse.py:47-52): ValueError for an empty group,
        a key outside [0, N) or a list that is not strictly ascending; ShapeError for a count
        above the row stride.  One HBM pass (fga_validate_mask) and a stream sync."""
        self.check_layout()
        t = torch()
        status = t.empty(2, dtype=t.int32, device=self.idx.device)
        rc, msg = _lib.call_rc("fga_validate_mask", ptr(self.idx), self.stride, ptr(self.counts),
                               self.batch * self.heads * self.num_groups, self.seq_len, ptr(status), stream_ptr())
        _raise_mask_status(rc, msg, int(status[0].item()) if rc != _lib.FGA_OK else 0)
        self.validated = True
        return self

    def tile_order(self, cfg: AttnConfig):
        """Longest-first claim order of the work tiles within each head (fga_tile_order), cached."""
        if self._order is None:
            t = torch()
            n = cfg.batch * cfg.heads * cfg.num_groups * (-(-cfg.group_size // 128))
            order = t.empty(n, dtype=t.int32, device=self.idx.device)
            _lib.call("fga_tile_order", ptr(self.counts), _lib.shape(*cfg.dims, cfg.group_size, cfg.scale), ptr(order),
                      stream_ptr())
            self._order = order
        return self._order

    def to_host(self) -> SparseIndexMask:
        idx = self.idx.cpu().numpy().reshape(-1, self.stride)
        cnt = self.counts.cpu().numpy().reshape(-1)
        flat = [np.sort(idx[r, : cnt[r]].astype(np.int64)) for r in range(idx.shape[0])]
        for a in flat:
            a.flags.writeable = False
        return SparseIndexMask._from_flat(self.batch, self.heads, self.seq_len, self.group_size, flat)


def _raise_mask_status(rc: int, msg: str, bits: int) -> None:
    """FGA_STATUS_* / return codes -> the reference's exceptions (sparse.py:47-52: ValueError)."""
    if rc == _lib.FGA_OK:
        return
    if bits & _lib.FGA_STATUS_EMPTY:
        raise ValueError("every group needs at least one key")
    if bits & _lib.FGA_STATUS_STRIDE:
        raise ShapeError("counts exceed the index row stride")
    if bits & _lib.FGA_STATUS_RANGE:
        raise ValueError(f"key index out of range ({msg})")
    if bits & _lib.FGA_STATUS_ORDER:
        raise ValueError(f"key lists must be sorted and unique ({msg})")
    _lib.check(rc, "mask check")


def _as_device_mask(mask, cfg: AttnConfig | None = None, device=None) -> DeviceIndexMask:
    """Device layout of any accepted mask; DeviceIndexMasks are layout-checked, and validated on
    the device once unless their producer guarantees the invariants."""
    if isinstance(mask, DeviceIndexMask):
        mask.check_layout(device)
        if not mask.validated:
            mask.validate()
        return mask
    if isinstance(mask, SparseIndexMask):
        return mask.to_device(device)
    if hasattr(mask, "keys_for") and hasattr(mask, "group_size"):  # a reference sliceattn mask
        lists = [[[mask.keys_for(b, h, g) for g in range(mask.num_groups)] for h in range(mask.heads)]
                 for b in range(mask.batch)]
        return SparseIndexMask(mask.batch, mask.heads, mask.seq_len, mask.group_size, lists).to_device(device)
    raise TypeError(f"unsupported mask type {type(mask).__name__}")


# ---------------------------------------------------------------- K1b compaction

def compact_keep(keep, group_size: int, scores=None, fill_sentinel: bool = False) -> DeviceIndexMask:
    """Keep bits [B, H, G, N] (uint8/bool, CUDA) -> DeviceIndexMask (fga_compact).

    Ascending positions per group, bit-exact with np.nonzero; with ``scores``
    an empty group keeps its first argmax (masks.py:75-91).  With
    ``fill_sentinel`` the idx tensor is exactly ``export_padded``'s layout."""
    t = torch()
    require_device()
    keep = as_device(keep, t.uint8)
    if keep.dim() != 4:
        raise ShapeError("keep must be [B, H, G, N]")
    b, h, g, n = keep.shape
    if g != -(-n // group_size):
        raise ShapeError(f"keep has {g} groups, group_size {group_size} implies {-(-n // group_size)}")
    sc = None
    if scores is not None:
        sc = as_device(scores, t.float32)
        if tuple(sc.shape) != tuple(keep.shape):
            raise ShapeError("scores must match keep")
    idx = t.empty((b, h, g, n), dtype=t.int32, device=keep.device)
    cnt = t.empty((b, h, g), dtype=t.int32, device=keep.device)
    _lib.call("fga_compact", ptr(keep), ptr(sc), b * h * g, n, ptr(idx), n, ptr(cnt), int(fill_sentinel), stream_ptr())
    # with scores an empty row keeps its argmax, so every list is non-empty, ascending, in range
    return DeviceIndexMask(b, h, n, group_size, idx, cnt, validated=sc is not None)


def compact_keep_bits(bits, group_size: int, seq_len: int, fill_sentinel: bool = False) -> DeviceIndexMask:
    """Bit-packed keep words [B, H, G, ceil(N/32)] (int32/uint32, CUDA) -> DeviceIndexMask
    (fga_compact_bits).  Same positions as compact_keep; no argmax fallback."""
    t = torch()
    require_device()
    bits = as_device(bits, t.int32)
    if bits.dim() != 4 or bits.shape[-1] != (seq_len + 31) // 32:
        raise ShapeError("bits must be [B, H, G, ceil(N/32)]")
    b, h, g, _ = bits.shape
    if g != -(-seq_len // group_size):
        raise ShapeError(f"bits have {g} groups, group_size {group_size} implies {-(-seq_len // group_size)}")
    idx = t.empty((b, h, g, seq_len), dtype=t.int32, device=bits.device)
    cnt = t.empty((b, h, g), dtype=t.int32, device=bits.device)
    _lib.call("fga_compact_bits", ptr(bits), b * h * g, seq_len, ptr(idx), seq_len, ptr(cnt), int(fill_sentinel),
              stream_ptr())
    return DeviceIndexMask(b, h, seq_len, group_size, idx, cnt)


# ---------------------------------------------------------------- K2 gather

@dataclass(frozen=True, eq=False)
class PackedTile:
    """Rows copied out of a source matrix, in ``source_indices`` order (sparse.py:87-92)."""

    rows: object
    source_indices: np.ndarray


def gather_rows(matrix, indices) -> PackedTile:
    """Copy the given rows (duplicates allowed), bitwise (sparse.py:95-108).

    Runs the K2 TMA gather4 producer on the device.  Row payloads of 128,
    256, 384 or 512 bytes are supported (bf16 D in {64..256}, fp32 D in
    {32, 64, 96, 128}); IndexError for indices outside [0, rows)."""
    t = torch()
    idx = np.asarray(indices.cpu() if is_torch(indices) else indices, dtype=np.int64)
    if idx.ndim != 1:
        raise ShapeError("indices must be one-dimensional")
    host = not is_torch(matrix)
    mat = t.from_numpy(np.ascontiguousarray(np.asarray(matrix))) if host else matrix
    if mat.dim() != 2:
        raise ShapeError("matrix must be [rows, D]")
    rows, d = mat.shape
    if idx.size and (idx.min() < 0 or idx.max() >= rows):
        raise IndexError(f"gather index out of range for {rows} rows")
    row_bytes = d * mat.element_size()
    if row_bytes % 128 != 0 or row_bytes > 512:
        raise NotImplementedError(f"gather_rows: {row_bytes}-byte rows unsupported (need 128/256/384/512)")
    dev = require_device()
    src = mat.to(f"cuda:{dev}").contiguous()
    words = src.view(t.int16).reshape(rows, row_bytes // 2)
    out = t.empty((idx.size, row_bytes // 2), dtype=t.int16, device=src.device)
    if idx.size:
        di = t.from_numpy(idx.astype(np.int32)).to(src.device)
        _lib.call("fga_gather_rows", ptr(words), rows, row_bytes // 2, ptr(di), idx.size, ptr(out), stream_ptr())
    res = out.view(src.dtype).reshape(idx.size, d)
    if host:
        res = res.cpu().numpy()
    idx.flags.writeable = False
    return PackedTile(rows=res, source_indices=idx)


# ---------------------------------------------------------------- attention

def chunk_trace(counts: np.ndarray, cfg: AttnConfig, chunk: int, kind: str = GATHER) -> list[TileEvent]:
    """TileEvents the chunk loop of sparse.py:145-154 would emit (one per <= chunk keys)."""
    ev = []
    counts = np.asarray(counts).reshape(cfg.batch, cfg.heads, cfg.num_groups)
    for b in range(cfg.batch):
        for h in range(cfg.heads):
            for g in range(cfg.num_groups):
                lo, hi = cfg.group_bounds(g)
                c = int(counts[b, h, g])
                ev.extend(TileEvent(b, h, g, hi - lo, min(chunk, c - s), kind) for s in range(0, c, chunk))
    return ev


def _check_qkv(cfg: AttnConfig, *ts):
    for t_ in ts:
        dims = tuple(t_.shape) if is_torch(t_) else tuple(getattr(t_, "dims", np.shape(getattr(t_, "data", t_))))
        if dims != cfg.dims:
            raise ShapeError(f"tensor dims {dims} do not match config {cfg.dims}")


_KERNEL_FLAGS = {"": 0, "dual": 0, "ws": _lib.FGA_ATTN_PER_TILE, "static": _lib.FGA_ATTN_STATIC,
                 "ws-static": _lib.FGA_ATTN_PER_TILE | _lib.FGA_ATTN_STATIC}


def attn_flags() -> int:
    """Kernel-selection flags for A/B runs: FGA_ATTN_KERNEL = ws (per-tile kernel for every
    shape), static (static tile stride), ws-static; default: dual kernel for 129..256-row
    groups, dynamic longest-first tile scheduling."""
    return _KERNEL_FLAGS[os.environ.get("FGA_ATTN_KERNEL", "")]


def _check_precision(cfg: AttnConfig, *ts) -> None:
    """The kernels compute on bf16 operands with fp32 accumulation.  That is the reference's
    precision='bf16' (inputs rounded on ingest, core.py:188-193); bf16 CUDA tensors are already
    there.  precision='full' on fp32 data asks for fp32 operands (1e-4 vs the dense
    oracle), which this path does not provide, so it is refused instead of silently rounded."""
    if cfg.precision == "bf16":
        return
    t = torch()
    if all(is_torch(x) and x.dtype == t.bfloat16 for x in ts):
        return
    raise NotImplementedError(
        "precision='full' needs fp32 operands; the B200 kernels compute with bf16 operands and fp32 "
        "accumulation -- use AttnConfig(..., precision='bf16') or pass bf16 CUDA tensors")


def _is_full(mask, dmask: DeviceIndexMask, cfg: AttnConfig) -> bool:
    """Every group lists every key (full_mask, sparse.py:206-213): attention over the listed keys is
    then dense attention, and the contiguous-chunk kernel (fga_dense_attn_fwd: TMA boxes, no index
    reads, no gather) computes it with the same chunk order and arithmetic.  Host masks answer from
    their counts; a device mask once per mask (one reduction + sync, cached)."""
    if os.environ.get("FGA_DENSE_DISPATCH", "1") == "0":
        return False
    cells = cfg.batch * cfg.heads * cfg.num_groups * cfg.seq_len
    if isinstance(mask, SparseIndexMask):
        return mask.total_indices == cells
    if dmask._full is None:
        dmask._full = bool(dmask.validated and int(dmask.counts.sum(dtype=torch().int64).item()) == cells)
    return dmask._full


def _run_dense(qd, kd, vd, cfg: AttnConfig, out_dtype, lse: bool):
    t = torch()
    o = t.empty(cfg.dims, dtype=out_dtype, device=qd.device)
    l = t.empty(cfg.dims[:3], dtype=t.float32, device=qd.device) if lse else None
    _lib.call("fga_dense_attn_fwd", ptr(qd), ptr(kd), ptr(vd), ptr(o),
              _lib.FGA_OUT_F32 if out_dtype == t.float32 else _lib.FGA_OUT_BF16, ptr(l),
              _lib.shape(*cfg.dims, cfg.group_size, cfg.scale), stream_ptr())
    return o, l


def _run_sparse(qd, kd, vd, dmask: DeviceIndexMask, cfg: AttnConfig, out_dtype, lse: bool, full: bool = False):
    if full:
        return _run_dense(qd, kd, vd, cfg, out_dtype, lse)
    t = torch()
    o = t.empty(cfg.dims, dtype=out_dtype, device=qd.device)
    l = t.empty(cfg.dims[:3], dtype=t.float32, device=qd.device) if lse else None
    flags = attn_flags()
    order = None if flags & _lib.FGA_ATTN_STATIC else dmask.tile_order(cfg)
    _lib.call("fga_sparse_attn_fwd_ex", ptr(qd), ptr(kd), ptr(vd), ptr(dmask.idx), dmask.stride, ptr(dmask.counts),
              ptr(o), _lib.FGA_OUT_F32 if out_dtype == t.float32 else _lib.FGA_OUT_BF16, ptr(l),
              _lib.shape(*cfg.dims, cfg.group_size, cfg.scale), 0, -1, ptr(order), None, flags, stream_ptr())
    return o, l


def sparse_attention(q, k, v, mask, cfg: AttnConfig, trace: list | None = None, chunk_size: int | None = None,
                     *, out_dtype=None, return_lse: bool = False):
    """Sparse attention over the masked key lists (sparse.py:111-156).

    ``mask`` is a SparseIndexMask, a DeviceIndexMask, or a
    ``masks.MaskBuilderConfig`` (the "threshold" form: the mask is built on
    the GPU from q and k first).  ``chunk_size`` only shapes the emitted
    ``trace``: the kernel always gathers 128-key chunks, and the result is
    chunking-invariant.  Host inputs return an fp32 AttnTensor;
    CUDA inputs return a CUDA tensor (bf16 unless ``out_dtype`` says otherwise),
    plus the natural-log normaliser per row when ``return_lse``."""
    _check_qkv(cfg, q, k, v)
    from .masks import MaskBuilderConfig, build_mask

    if isinstance(mask, MaskBuilderConfig):
        mask = build_mask(q, k, cfg, mask, device_result=True)
    mask.check_compatible(cfg)
    chunk = cfg.group_size if chunk_size is None else chunk_size
    if chunk < 1 or chunk > cfg.group_size:
        raise ValueError(f"chunk_size must be in [1, {cfg.group_size}]")
    t = torch()
    host = not is_torch(q)
    _check_precision(cfg, q, k, v)
    qd, kd, vd = as_device_bf16(q), as_device_bf16(k), as_device_bf16(v)
    dmask = _as_device_mask(mask, cfg, qd.device.index)
    dt = t.float32 if host else (out_dtype or t.bfloat16)
    o, l = _run_sparse(qd, kd, vd, dmask, cfg, dt, return_lse, full=_is_full(mask, dmask, cfg))
    if trace is not None:
        counts = mask.counts() if isinstance(mask, SparseIndexMask) else dmask.counts.cpu().numpy()
        trace.extend(chunk_trace(counts, cfg, chunk, GATHER))
    if host:
        out = o.cpu().numpy()
        if not np.isfinite(out).all():
            raise NumericError("non-finite attention output")
        res = AttnTensor(out)
        return (res, l.cpu().numpy()) if return_lse else res
    return (o, l) if return_lse else o


def masked_dense_attention(q, k, v, mask, cfg: AttnConfig):
    """oracle.py:55-82 semantics (softmax over exactly the listed keys) -- on the
    device this is the same kernel as sparse_attention."""
    return sparse_attention(q, k, v, mask, cfg)


# ---------------------------------------------------------------- mask helpers

def mask_density(mask) -> float:
    """Retained fraction of (group, key) pairs (sparse.py:159-162)."""
    total = mask.batch * mask.heads * mask.num_groups * mask.seq_len
    return mask.total_indices / total


def export_padded(mask):
    """[B, H, G, N] int32, list prefix then -1 (sparse.py:165-175).

    Host mask -> ndarray; DeviceIndexMask -> CUDA tensor (the device layout
    with its tail forced to -1)."""
    if isinstance(mask, DeviceIndexMask):
        t = torch()
        col = t.arange(mask.stride, device=mask.idx.device, dtype=t.int32)
        out = t.where(col < mask.counts[..., None], mask.idx, t.full_like(mask.idx, -1))
        return out[..., : mask.seq_len].contiguous()
    if not isinstance(mask, SparseIndexMask):
        mask = _as_device_mask(mask).to_host()
    return _padded_host(mask)


def import_padded(padded, group_size: int):
    """Inverse of export_padded (sparse.py:178-203); rejects interior sentinels.
    A CUDA tensor gives a validated DeviceIndexMask, an array a SparseIndexMask."""
    if is_torch(padded) and padded.is_cuda:
        t = torch()
        if padded.dim() != 4:
            raise ShapeError(f"expected [B, H, G, N] array, got shape {tuple(padded.shape)}")
        b, h, g, n = padded.shape
        if g != -(-n // group_size):
            raise ShapeError(f"padded array has {g} groups, group_size {group_size} implies {-(-n // group_size)}")
        p = padded.to(t.int32).contiguous()
        used = p >= 0
        cnt = used.sum(-1, dtype=t.int32)
        col = t.arange(n, device=p.device, dtype=t.int32)
        if bool((used != (col < cnt[..., None])).any().item()):
            raise ValueError("sentinel slots must trail the key indices")
        # the host path builds a SparseIndexMask, whose np.unique sorts and deduplicates every
        # list (sparse.py:46); do the same on the device so both give the same mask
        big = t.iinfo(t.int32).max
        srt = t.where(used, p, t.full_like(p, big)).sort(dim=-1).values
        dup = t.zeros_like(used)
        dup[..., 1:] = srt[..., 1:] == srt[..., :-1]
        srt = t.where(dup, t.full_like(srt, big), srt).sort(dim=-1).values
        live = srt != big
        cnt = live.sum(-1, dtype=t.int32)
        srt = t.where(live, srt, t.full_like(srt, -1)).contiguous()
        return DeviceIndexMask(b, h, n, group_size, srt, cnt).validate()
    arr = np.asarray(padded)
    if arr.ndim != 4:
        raise ShapeError(f"expected [B, H, G, N] array, got shape {arr.shape}")
    b, h, g, n = arr.shape
    if g != -(-n // group_size):
        raise ShapeError(f"padded array has {g} groups, group_size {group_size} implies {-(-n // group_size)}")
    rows = arr.reshape(-1, n)
    lists = []
    for r in rows:
        used = r >= 0
        c = int(used.sum())
        if not used[:c].all():
            raise ValueError("sentinel slots must trail the key indices")
        lists.append(r[:c])
    nested = [[lists[(bb * h + hh) * g:(bb * h + hh + 1) * g] for hh in range(h)] for bb in range(b)]
    return SparseIndexMask(b, h, n, group_size, nested)


def full_mask(cfg: AttnConfig) -> SparseIndexMask:
    """Every key for every group (sparse.py:206-213)."""
    keys = np.arange(cfg.seq_len, dtype=np.int64)
    keys.flags.writeable = False
    flat = [keys] * (cfg.batch * cfg.heads * cfg.num_groups)
    return SparseIndexMask._from_flat(cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size, flat)


def random_mask(cfg: AttnConfig, density: float, seed: int = 0) -> SparseIndexMask:
    """Uniformly random mask, max(1, round(d*N)) keys per group, drawn from the
    same Philox stream as the reference (sparse.py:216-232) so masks agree
    key for key.  Host-side generation; see random_mask_device for HBM masks."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    rng = np.random.Generator(np.random.Philox(seed))
    count = max(1, round(density * cfg.seq_len))
    flat = []
    for _ in range(cfg.batch * cfg.heads * cfg.num_groups):
        a = np.sort(rng.choice(cfg.seq_len, size=count, replace=False).astype(np.int64))
        a.flags.writeable = False
        flat.append(a)
    return SparseIndexMask._from_flat(cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size, flat)


def random_mask_device(cfg: AttnConfig, density: float, seed: int = 0, fill_sentinel: bool = False) -> DeviceIndexMask:
    """Device-generated mask with the same count rule (fga_random_keep: a
    counter-based hash picks exactly max(1, round(d*N)) keys per group), then
    K1b compaction.  Not the reference's Philox stream -- for benchmarks."""
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    t = torch()
    dev = require_device()
    count = max(1, round(density * cfg.seq_len))
    rows = cfg.batch * cfg.heads * cfg.num_groups
    keep = t.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=t.uint8, device=f"cuda:{dev}")
    _lib.call("fga_random_keep", rows, cfg.seq_len, count, int(seed) & 0xFFFFFFFFFFFFFFFF, ptr(keep), stream_ptr())
    mask = compact_keep(keep, cfg.group_size, None, fill_sentinel)
    mask.validated = True  # exactly max(1, round(d*N)) distinct keys per row
    return mask


def mask_jaccard(a, b) -> float:
    """Jaccard overlap of two masks' (group, key) pairs (sparse.py:235-250); host utility."""
    if (a.batch, a.heads, a.seq_len, a.group_size) != (b.batch, b.heads, b.seq_len, b.group_size):
        raise ShapeError("masks have different dims")
    ha = a if isinstance(a, SparseIndexMask) else a.to_host()
    hb = b if isinstance(b, SparseIndexMask) else b.to_host()
    inter = union = 0
    for x, y in zip(ha._lists, hb._lists):
        c = np.intersect1d(x, y, assume_unique=True).size
        inter += c
        union += x.size + y.size - c
    return inter / union
