"""Host-resident inputs: overlap PCIe transfers with the kernels.

``sparse_attention_host(q, k, v, keep_bits, cfg)`` takes pinned CPU tensors
(bf16 Q/K/V [B,H,N,D], uint32 bit-packed slice mask [B,H,G,ceil(N/32)]) and
fills a pinned CPU output.  The (b,h) heads are cut into slabs; slab s+1's
H2D copy (copy engine), slab s's K1b bit compaction + attention (SMs) and
slab s-1's D2H copy run concurrently on three streams, so the step costs
about max(H2D, compute, D2H) instead of their sum.  Heads are independent
(sparse.py:138-155), so slabs need no exchange.  The call is stream-ordered
after the caller's current stream and makes that stream wait for the last
D2H, so CUDA events on the caller's stream time the whole transfer+compute.
"""

from __future__ import annotations

from . import _lib
from ._device import ptr, require_device, torch
from .core import AttnConfig, ShapeError

__all__ = ["pack_keep_bits", "HostPipeline", "sparse_attention_host"]


def pack_keep_bits(keep):
    """uint8/bool keep [..., N] (CUDA) -> uint32 bits [..., ceil(N/32)] (fga_pack_bits)."""
    t = torch()
    require_device()
    keep = keep.to(t.uint8).contiguous()
    n = keep.shape[-1]
    rows = keep.numel() // n
    words = (n + 31) // 32
    bits = t.empty(tuple(keep.shape[:-1]) + (words,), dtype=t.int32, device=keep.device)
    _lib.call("fga_pack_bits", ptr(keep), rows, n, ptr(bits), t.cuda.current_stream().cuda_stream)
    return bits


class HostPipeline:
    """Device buffers + streams for one problem shape (reused across calls)."""

    def __init__(self, cfg: AttnConfig, slabs: int = 4, device=None, tail: bool = True, tail_parts: int = 2):
        t = torch()
        self.dev = require_device(device)
        self.cfg = cfg
        bh = cfg.batch * cfg.heads
        slabs = max(1, min(slabs, bh))
        # The step costs about sum(H2D) + compute + D2H of the LAST slab (everything else hides
        # under the next slab's upload), so with a short tail the last slab is a single head and
        # the other heads are split evenly over the remaining slabs.
        sizes = []
        if tail and slabs > 1 and bh > slabs:
            base, extra = divmod(bh - 1, slabs - 1)
            sizes = [base + (1 if s < extra else 0) for s in range(slabs - 1)] + [1]
        else:
            base, extra = divmod(bh, slabs)
            sizes = [base + (1 if s < extra else 0) for s in range(slabs)]
        self.ranges, h0 = [], 0
        for sz in sizes:
            self.ranges.append((h0, h0 + sz))
            h0 += sz
        # With a one-head tail, that head's K/V/bits go up first and its query groups in
        # `tail_parts` runs (fga_sparse_attn_fwd_tiles), so only the last run's Q upload, one
        # wave of tiles and the last run's D2H remain after the bulk of the PCIe traffic.
        g = cfg.num_groups
        parts = max(1, min(tail_parts, g)) if (sizes and sizes[-1] == 1 and len(sizes) > 1) else 1
        self.tail_groups = [(g * i // parts, g * (i + 1) // parts) for i in range(parts)]
        n, d, g = cfg.seq_len, cfg.head_dim, cfg.num_groups
        self.words = (n + 31) // 32
        kw = dict(device=f"cuda:{self.dev}")
        self.q = t.empty((bh, n, d), dtype=t.bfloat16, **kw)
        self.k = t.empty_like(self.q)
        self.v = t.empty_like(self.q)
        self.o = t.empty_like(self.q)
        self.bits = t.empty((bh, g, self.words), dtype=t.int32, **kw)
        self.idx = t.empty((bh, g, n), dtype=t.int32, **kw)
        self.counts = t.empty((bh, g), dtype=t.int32, **kw)
        # mask violations seen by the kernels (FGA_STATUS_* bits), read back once per call
        self.status = t.zeros(2, dtype=t.int32, **kw)
        self.status_host = t.zeros(2, dtype=t.int32).pin_memory()
        self.s_h2d = t.cuda.Stream(self.dev)
        self.s_cmp = t.cuda.Stream(self.dev)
        self.s_d2h = t.cuda.Stream(self.dev)

    def __call__(self, q, k, v, keep_bits, out, check: bool = True):
        t = torch()
        cfg = self.cfg
        bh, n, d, g = cfg.batch * cfg.heads, cfg.seq_len, cfg.head_dim, cfg.num_groups
        hq, hk, hv, ho = (x.view(bh, n, d) for x in (q, k, v, out))
        hb = keep_bits.view(bh, g, self.words)
        caller = t.cuda.current_stream(self.dev)
        start = caller.record_event()
        for s_ in (self.s_h2d, self.s_cmp, self.s_d2h):
            s_.wait_event(start)
        with t.cuda.stream(self.s_cmp):
            self.status.zero_()
        st = ptr(self.status)
        last = None
        m = cfg.group_size
        tpg = -(-m // 128)  # work tiles per group
        for si, (h0, h1) in enumerate(self.ranges):
            if si == len(self.ranges) - 1 and len(self.tail_groups) > 1:
                with t.cuda.stream(self.s_h2d):
                    for dst, src in ((self.bits, hb), (self.k, hk), (self.v, hv)):
                        dst[h0:h1].copy_(src[h0:h1], non_blocking=True)
                sh = _lib.shape(1, 1, n, d, m, cfg.scale)
                cs = self.s_cmp.cuda_stream
                for g0, g1 in self.tail_groups:
                    r0, r1 = g0 * m, min(g1 * m, n)
                    with t.cuda.stream(self.s_h2d):
                        self.q[h0, r0:r1].copy_(hq[h0, r0:r1], non_blocking=True)
                        ev_in = self.s_h2d.record_event()
                    self.s_cmp.wait_event(ev_in)
                    _lib.call("fga_compact_bits", ptr(self.bits[h0, g0]), g1 - g0, n, ptr(self.idx[h0, g0]), n,
                              ptr(self.counts[h0, g0]), 0, cs)
                    _lib.call("fga_sparse_attn_fwd_ex", ptr(self.q[h0]), ptr(self.k[h0]), ptr(self.v[h0]),
                              ptr(self.idx[h0]), n, ptr(self.counts[h0]), ptr(self.o[h0]), _lib.FGA_OUT_BF16, None,
                              sh, g0 * tpg, g1 * tpg, None, st, 0, cs)
                    ev_c = self.s_cmp.record_event()
                    self.s_d2h.wait_event(ev_c)
                    with t.cuda.stream(self.s_d2h):
                        ho[h0, r0:r1].copy_(self.o[h0, r0:r1], non_blocking=True)
                        last = self.s_d2h.record_event()
                continue
            with t.cuda.stream(self.s_h2d):
                for dst, src in ((self.bits, hb), (self.q, hq), (self.k, hk), (self.v, hv)):
                    dst[h0:h1].copy_(src[h0:h1], non_blocking=True)
                ev_in = self.s_h2d.record_event()
            self.s_cmp.wait_event(ev_in)
            rows = (h1 - h0) * g
            sh = _lib.shape(1, h1 - h0, n, d, cfg.group_size, cfg.scale)
            cs = self.s_cmp.cuda_stream
            _lib.call("fga_compact_bits", ptr(self.bits[h0]), rows, n, ptr(self.idx[h0]), n, ptr(self.counts[h0]), 0, cs)
            _lib.call("fga_sparse_attn_fwd_ex", ptr(self.q[h0]), ptr(self.k[h0]), ptr(self.v[h0]), ptr(self.idx[h0]),
                      n, ptr(self.counts[h0]), ptr(self.o[h0]), _lib.FGA_OUT_BF16, None, sh, 0, -1, None, st, 0, cs)
            ev_c = self.s_cmp.record_event()
            self.s_d2h.wait_event(ev_c)
            with t.cuda.stream(self.s_d2h):
                ho[h0:h1].copy_(self.o[h0:h1], non_blocking=True)
                last = self.s_d2h.record_event()
        # the status word follows the last attention launch on s_cmp
        done_cmp = self.s_cmp.record_event()
        self.s_d2h.wait_event(done_cmp)
        with t.cuda.stream(self.s_d2h):
            self.status_host.copy_(self.status, non_blocking=True)
            last = self.s_d2h.record_event()
        caller.wait_event(last)
        if check:
            # an empty slice-mask row has no softmax denominator: the reference raises
            # (sparse.py:47-48 on the mask, tiled.py:75-76 in finalize); the kernels only flag it
            last.synchronize()
            bits = int(self.status_host[0])
            if bits & _lib.FGA_STATUS_EMPTY:
                raise ValueError("every group needs at least one key (an all-zero keep_bits row)")
        return out


_pipes: dict = {}


def sparse_attention_host(q, k, v, keep_bits, cfg: AttnConfig, out=None, slabs: int = 5, tail: bool = True,
                          tail_parts: int = 2, check: bool = True):
    """FG-Attn from pinned host buffers (see module doc).  Returns the pinned host output.
    With ``check`` (default) the call waits for the step and raises ValueError when a slice-mask
    row keeps no key (sparse.py:47-48); with ``check=False`` it returns at once and the caller
    synchronises the current stream before reading the output."""
    t = torch()
    for x in (q, k, v):
        if tuple(x.shape) != cfg.dims:
            raise ShapeError(f"tensor dims {tuple(x.shape)} do not match config {cfg.dims}")
        if x.dtype != t.bfloat16 or x.is_cuda:
            raise ShapeError("q, k, v must be host bf16 tensors (pinned for overlap)")
    expect = (cfg.batch, cfg.heads, cfg.num_groups, (cfg.seq_len + 31) // 32)
    if tuple(keep_bits.shape) != expect:
        raise ShapeError(f"keep_bits must be {expect}, got {tuple(keep_bits.shape)}")
    key = (cfg, slabs, tail, tail_parts, require_device())
    if key not in _pipes:
        _pipes[key] = HostPipeline(cfg, slabs, tail=tail, tail_parts=tail_parts)
    if out is None:
        out = t.empty(cfg.dims, dtype=t.bfloat16, pin_memory=True)
    return _pipes[key](q, k, v, keep_bits, out, check)
