"""Sparsity analyzers (masks.py:153-184).

CPU: the oracle restatement against the reference itself (skipped where /root/reference is
absent, e.g. on the GPU box) and the SPEC.md:327 constructed-map example.
GPU: block/slice sparsity from an explicit map and from Q, K (no N x N map) against the oracle."""

import os
import sys

import numpy as np
import pytest

import oracle
from conftest import cuda_ok

REF = "/root/reference/pkg/src/sliceattn"


def block_diag_map(n=128):
    # two 64x64 blocks of mass on the diagonal (each row uniform over its block)
    a = np.zeros((1, 1, n, n), np.float32)
    a[0, 0, :64, :64] = 1 / 64
    a[0, 0, 64:, 64:] = 1 / 64
    return a


def test_oracle_spec_example():
    assert oracle.block_sparsity(block_diag_map(), 64, 0.5 / 128) == 0.5


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_oracle_matches_reference_analyzers():
    sys.path.insert(0, os.path.dirname(REF))
    from sliceattn import core as rcore, masks as rmasks

    rng = np.random.default_rng(3)
    for n, m in ((200, 64), (256, 128)):
        s = rng.standard_normal((1, 2, n, n)) * 3
        a = (np.exp(s) / np.exp(s).sum(-1, keepdims=True)).astype(np.float32)
        amap = rcore.AttnMap(a)
        for block in (16, 32, 64):
            for tau in (0.5 / n, 2.0 / n):
                assert oracle.block_sparsity(a, block, tau) == rmasks.block_sparsity(amap, block, tau)
        for prec in ("full", "bf16"):
            cfg = rcore.AttnConfig(1, 2, n, 32, group_size=m, precision=prec)
            assert oracle.slice_sparsity(a, m, 1.0 / n, prec) == rmasks.slice_sparsity(amap, cfg, 1.0 / n)


@pytest.mark.gpu
def test_gpu_analyzers_match_oracle():
    if not cuda_ok():
        pytest.skip("needs a CUDA device")
    import paper_2509_16518_b200 as fga

    assert fga.block_sparsity(block_diag_map(), 64, 0.5 / 128) == 0.5
    rng = np.random.default_rng(5)
    b, h, n, d = 1, 2, 384, 64
    q = oracle.bf16_round(2.0 * rng.standard_normal((b, h, n, d)).astype(np.float32))
    k = oracle.bf16_round(rng.standard_normal((b, h, n, d)).astype(np.float32))
    a = oracle.attention_map(q, k, precision="full")
    vals = []
    for block in (16, 32, 64, 128):
        want = oracle.block_sparsity(a, block, 1.0 / n)
        assert fga.block_sparsity(a, block, 1.0 / n) == want
        got_qk = fga.block_sparsity_qk(q, k, fga.AttnConfig(b, h, n, d), block, 1.0 / n)
        tiles = (-(-n // block)) ** 2
        assert abs(got_qk - want) <= 2.0 / tiles       # fused fp32 scores may flip a tile at tau
        vals.append(want)
    assert vals == sorted(vals, reverse=True)          # SPEC.md:341 granularity monotonicity
    for prec in ("full", "bf16"):
        cfg = fga.AttnConfig(b, h, n, d, group_size=128, precision=prec)
        want = oracle.slice_sparsity(a, 128, 1.0 / n, prec)
        assert fga.slice_sparsity(a, cfg, 1.0 / n) == want
        assert abs(fga.slice_sparsity_qk(q, k, cfg, 1.0 / n) - want) <= 1e-3
