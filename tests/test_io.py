"""FGT1 / FGM1 file formats (paper_2509_16518_b200/io.py).

CPU: byte-level round trips, the spec's negative cases (bad magic, truncated payload,
dimension overflow) and the committed fixture (tests/golden/lens_ragged.fgm1, the
reference-generated lens_ragged mask encoded by tests/golden/make_fgm1.py).
GPU: the device decoder (fga_fgm1_unpack) equals the host decode, bit for bit."""

import hashlib
import os

import numpy as np
import pytest

import oracle
from conftest import cuda_ok
from paper_2509_16518_b200 import AttnConfig, io as fio, random_mask

FIXTURE = os.path.join(os.path.dirname(__file__), "golden", "lens_ragged.fgm1")
FIXTURE_SHA = "8396614c6f1d3683b71d488f073f5848b1ddaa04cc410f30969cd22249ed5474"


def test_tensor_round_trip_bitwise(tmp_path):
    x = np.random.default_rng(0).standard_normal((2, 3, 17, 8)).astype(np.float32)
    p = str(tmp_path / "t.fgt1")
    fio.write_tensor(p, x)
    y = fio.read_tensor(p).data
    assert y.dtype == np.float32 and y.shape == x.shape and y.tobytes() == x.tobytes()
    assert fio.encode_tensor(y) == fio.encode_tensor(x)
    s = np.random.default_rng(1).standard_normal((1, 2, 16, 16))
    mp = (np.exp(s) / np.exp(s).sum(-1, keepdims=True) * 0.999).astype(np.float32)   # a valid AttnMap
    fio.write_map(str(tmp_path / "m.fgt1"), mp)
    assert fio.read_map(str(tmp_path / "m.fgt1")).data.tobytes() == mp.tobytes()


def test_tensor_errors():
    buf = fio.encode_tensor(np.ones((4, 5), np.float32))
    with pytest.raises(fio.FormatError):
        fio.decode_tensor(b"XXXX" + buf[4:])
    with pytest.raises(fio.CorruptionError):
        fio.decode_tensor(buf[:-1])                      # truncated by one byte
    with pytest.raises(fio.CorruptionError):
        fio.decode_tensor(buf + b"\0\0\0\0")             # trailing payload
    huge = bytearray(buf)
    huge[12:20] = (2 ** 40).to_bytes(8, "little")        # dimension overflow vs payload
    with pytest.raises(fio.CorruptionError):
        fio.decode_tensor(bytes(huge))


def test_mask_round_trip_identity(tmp_path):
    cfg = AttnConfig(2, 3, 1000, 64, group_size=100)
    mask = random_mask(cfg, 0.37, seed=5)
    p = str(tmp_path / "m.fgm1")
    fio.write_mask(p, mask)
    back = fio.read_mask(p)
    assert (back.batch, back.heads, back.seq_len, back.group_size) == (2, 3, 1000, 100)
    for b in range(2):
        for h in range(3):
            for g in range(cfg.num_groups):
                assert np.array_equal(back.keys_for(b, h, g), mask.keys_for(b, h, g))
    assert fio.encode_mask(back) == open(p, "rb").read()       # encode(decode(x)) == x


def test_mask_errors():
    cfg = AttnConfig(1, 1, 256, 64)
    buf = fio.encode_mask(random_mask(cfg, 0.5, seed=1))
    with pytest.raises(fio.FormatError):
        fio.decode_mask(b"FGT1" + buf[4:])
    with pytest.raises(fio.CorruptionError):
        fio.decode_mask(buf[:-4])
    with pytest.raises(fio.CorruptionError):
        fio.decode_mask(buf + b"\1\0\0\0")
    bad = bytearray(buf)
    first = int.from_bytes(bad[48:52], "little")
    bad[52 + 4 * (first - 1):52 + 4 * first] = (9999).to_bytes(4, "little")   # index >= N
    with pytest.raises(fio.CorruptionError):
        fio.decode_mask(bytes(bad))
    huge = bytearray(buf)
    huge[8:16] = (1 << 40).to_bytes(8, "little")   # B = 2^40: rejected before any allocation
    with pytest.raises(fio.CorruptionError):
        fio.decode_mask(bytes(huge))


def test_committed_fixture_decodes_to_reference_lists(golden):
    raw = open(FIXTURE, "rb").read()
    assert hashlib.sha256(raw).hexdigest() == FIXTURE_SHA
    g = golden("lens_ragged")
    mask = fio.decode_mask(raw)
    ref = g.lists()
    got = [mask.keys_for(b, h, gg) for b in range(mask.batch) for h in range(mask.heads)
           for gg in range(-(-mask.seq_len // mask.group_size))]
    assert len(got) == len(ref) and all(np.array_equal(a, b) for a, b in zip(got, ref))
    assert np.array_equal(oracle.lists_to_padded(got, mask.batch, mask.heads, len(got) // (mask.batch * mask.heads),
                                                 mask.seq_len), g["padded"])


@pytest.mark.gpu
def test_device_decoder_matches_host_decode():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import torch

    from paper_2509_16518_b200 import export_padded

    raw = open(FIXTURE, "rb").read()
    host = fio.decode_mask(raw)
    dm = fio.read_mask_device(raw, fill_sentinel=True)
    assert np.array_equal(dm.idx.cpu().numpy(), export_padded(host))
    cfg = AttnConfig(1, 4, 3000, 128)
    mask = random_mask(cfg, 0.21, seed=9)
    dm2 = fio.read_mask_device(fio.encode_mask(mask))
    torch.cuda.synchronize()
    for h in range(4):
        for g in range(cfg.num_groups):
            c = int(dm2.counts[0, h, g])
            assert np.array_equal(dm2.idx[0, h, g, :c].cpu().numpy(), mask.keys_for(0, h, g))
