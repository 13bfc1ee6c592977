"""K2 of the hot path in isolation: the attention kernel's own cp.async producer warps
(attn_ws.cu producer_half) fill the K/V ring slots for one key list, and every slot is copied
back out of the 128B swizzle (fga_gather_ring_probe).  The packed rows must equal
gather_rows (/root/reference/pkg/src/sliceattn/sparse.py:95-108) bitwise, with the tail of the
last chunk zero-filled -- the rows the tensor core reads for S = Q K^T and O += P V.
GPU only."""

import pytest

from conftest import cuda_ok

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not cuda_ok():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2509_16518_b200 as fga  # noqa: E402
from paper_2509_16518_b200 import _lib  # noqa: E402


def _probe(k, v, idx, count, stride=None):
    n, d = k.shape
    stride = stride or max(1, idx.numel())
    c = min(count, stride)
    rows = 128 * (-(-c // 128))
    ok = torch.full((max(rows, 1), d), float("nan"), device="cuda").to(torch.bfloat16)
    ov = torch.full((max(rows, 1), d), float("nan"), device="cuda").to(torch.bfloat16)
    cnt = torch.tensor([count], dtype=torch.int32, device="cuda")
    _lib.call("fga_gather_ring_probe", k.data_ptr(), v.data_ptr(), n, d, idx.data_ptr(), stride, cnt.data_ptr(),
              ok.data_ptr(), ov.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return ok[:rows], ov[:rows], c


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("count", [1, 77, 128, 129, 1000, 1843])
def test_ring_slots_equal_gather_rows_bitwise(d, count):
    # 1843 keys = 15 chunks: every one of the 3 + 3 ring slots is reused five times
    n = 4096
    g = torch.Generator(device="cuda").manual_seed(count + d)
    k = torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16)
    keys = torch.sort(torch.randperm(n, device="cuda", generator=g)[:count]).values.to(torch.int32)
    ok, ov, c = _probe(k, v, keys, count)
    ref_k = fga.gather_rows(k, keys).rows  # the K2 primitive itself (TMA gather4), bitwise = k[keys]
    assert torch.equal(ref_k.view(torch.int16), k[keys.long()].view(torch.int16))
    assert torch.equal(ok[:c].view(torch.int16), ref_k.view(torch.int16))
    assert torch.equal(ov[:c].view(torch.int16), v[keys.long()].view(torch.int16))
    assert not ok[c:].view(torch.int16).any() and not ov[c:].view(torch.int16).any()  # zero-filled tail


def test_ring_any_order_duplicates_and_stride_clamp():
    n, d = 3000, 128
    k = torch.randn(n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(n, d, device="cuda").to(torch.bfloat16)
    keys = torch.tensor([5, 2999, 5, 0, 1234] * 60, dtype=torch.int32, device="cuda")  # unsorted, repeated
    ok, ov, c = _probe(k, v, keys, 300)
    assert torch.equal(ok[:c].view(torch.int16), k[keys.long()].view(torch.int16))
    # a count above the list stride is clamped to the stride (the kernel never reads the next list)
    ok2, _, c2 = _probe(k, v, keys, 10_000, stride=200)
    assert c2 == 200 and torch.equal(ok2[:200].view(torch.int16), k[keys[:200].long()].view(torch.int16))


def test_ring_out_of_range_keys_are_clamped_not_read_out_of_bounds():
    n, d = 1000, 64
    k = torch.randn(n, d, device="cuda").to(torch.bfloat16)
    v = torch.randn(n, d, device="cuda").to(torch.bfloat16)
    keys = torch.tensor([3, -7, 1000, 1 << 30, 999], dtype=torch.int32, device="cuda")
    ok, _, c = _probe(k, v, keys, 5)
    clamped = torch.tensor([3, 999, 999, 999, 999], device="cuda")  # min(unsigned key, n - 1)
    assert torch.equal(ok[:c].view(torch.int16), k[clamped].view(torch.int16))
