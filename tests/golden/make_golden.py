"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):  ``python tests/golden/make_golden.py``.  It imports
``sliceattn`` from ``/root/reference/pkg/src`` and writes one compressed
``.npz`` per case next to this script.  Q/K/V are not stored: they are the
reference's own ``new_tensor(cfg, 'gaussian', seed)`` draws (core.py:150-167),
which the tests regenerate with NumPy's Philox and verify against the
SHA-256 recorded here.

Every case records: config, the mask as ``export_padded`` indices
(sparse.py:165-175), the reference ``sparse_attention`` output
(sparse.py:111-156) and, where cheap, ``masked_dense_attention``
(oracle.py:55-82), plus builder inputs/outputs for the mask builders
(masks.py:94-150) and ``count_flops`` fields (perfmodel.py:92-110).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import sliceattn.core as core
    import sliceattn.masks as masks
    import sliceattn.oracle as oracle
    import sliceattn.perfmodel as perfmodel
    import sliceattn.sparse as sparse
    import sliceattn.tiled as tiled
    return core, sparse, oracle, masks, perfmodel, tiled


core, sparse, oracle, masks, perfmodel, tiled = _ref()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def qkv(cfg, seeds=(1, 2, 3), qmul=1.0):
    q = core.new_tensor(cfg, "gaussian", seed=seeds[0])
    if qmul != 1.0:
        q = core.AttnTensor(q.data * np.float32(qmul))
    k = core.new_tensor(cfg, "gaussian", seed=seeds[1])
    v = core.new_tensor(cfg, "gaussian", seed=seeds[2])
    return q, k, v


def save(name, cfg, mask, q, k, v, extra=None, outputs=True, seeds=(1, 2, 3), qmul=1.0):
    payload = {
        "cfg": np.array(json.dumps(dict(
            batch=cfg.batch, heads=cfg.heads, seq_len=cfg.seq_len,
            head_dim=cfg.head_dim, group_size=cfg.group_size,
            scale=cfg.scale, precision=cfg.precision,
            seeds=list(seeds), qmul=qmul,
            numpy=np.__version__))),
        "q_sha": np.array(sha(q.data)),
        "k_sha": np.array(sha(k.data)),
        "v_sha": np.array(sha(v.data)),
    }
    if mask is not None:
        padded = sparse.export_padded(mask)
        payload["padded"] = padded.astype(np.int16 if cfg.seq_len < 32768 else np.int32)
        payload["counts"] = (padded >= 0).sum(axis=3).astype(np.int32)
        rep = perfmodel.count_flops(cfg, mask)
        payload["count_flops"] = np.array(json.dumps(rep.as_dict()))
        payload["density"] = np.array(sparse.mask_density(mask))
        if outputs:
            trace = []
            out = sparse.sparse_attention(q, k, v, mask, cfg, trace=trace)
            payload["sparse_out"] = out.data
            payload["trace_len"] = np.array(len(trace))
            payload["trace_keys"] = np.array([e.keys for e in trace], dtype=np.int32)
            if cfg.seq_len <= 1024:
                payload["masked_dense_out"] = oracle.masked_dense_attention(
                    q, k, v, mask, cfg).data
    for key, val in (extra or {}).items():
        payload[key] = val
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **payload)
    print(name, {k: getattr(v, "shape", None) for k, v in payload.items()})


def custom_mask(cfg, lens, seed):
    """Lists with prescribed lengths (cycled), random keys."""
    rng = np.random.default_rng(seed)
    it = 0
    lists = []
    for _b in range(cfg.batch):
        per_b = []
        for _h in range(cfg.heads):
            per_h = []
            for _g in range(cfg.num_groups):
                n_keys = lens[it % len(lens)]
                it += 1
                per_h.append(rng.choice(cfg.seq_len, size=n_keys, replace=False))
            per_b.append(per_h)
        lists.append(per_b)
    return sparse.SparseIndexMask(cfg.batch, cfg.heads, cfg.seq_len, cfg.group_size, lists)


def main():
    # c1: BASELINE.json configs[0], SURVEY.md section 8(d) parity config.
    cfg = core.AttnConfig(1, 2, 4096, 64, precision="bf16")
    q, k, v = qkv(cfg)
    save("c1_random30", cfg, sparse.random_mask(cfg, 0.3, seed=0), q, k, v)

    # ragged N (N % 128 = 104), short last group.
    cfg = core.AttnConfig(1, 2, 1000, 64, precision="bf16")
    q, k, v = qkv(cfg, (11, 12, 13))
    save("ragged_n1000", cfg, sparse.random_mask(cfg, 0.2, seed=5), q, k, v, seeds=(11, 12, 13))

    # D = 128, Wan head dim, two batches.
    cfg = core.AttnConfig(2, 2, 640, 128, precision="bf16")
    q, k, v = qkv(cfg, (21, 22, 23))
    save("d128_b2", cfg, sparse.random_mask(cfg, 0.25, seed=7), q, k, v, seeds=(21, 22, 23))

    # full mask == dense; also keep the dense outputs.
    cfg = core.AttnConfig(1, 1, 384, 64, precision="bf16")
    q, k, v = qkv(cfg, (31, 32, 33))
    dense = oracle.dense_attention(q, k, v, cfg).data
    flash = tiled.flash_attention(q, k, v, cfg).data
    save("full_n384", cfg, sparse.full_mask(cfg), q, k, v, seeds=(31, 32, 33),
         extra={"dense_out": dense, "flash_out": flash})

    # ragged list lengths: 1, 3 (mod 4), 127, 129 (== 1 mod 128), 257, 255.
    cfg = core.AttnConfig(1, 2, 768, 64, precision="bf16")
    q, k, v = qkv(cfg, (41, 42, 43))
    save("lens_ragged", cfg, custom_mask(cfg, [1, 3, 127, 129, 257, 255, 5, 2], 99),
         q, k, v, seeds=(41, 42, 43))

    # group_size != 128 (M = 64, N = 300 -> 5 groups, last has 44 rows).
    cfg = core.AttnConfig(1, 1, 300, 64, group_size=64, precision="bf16")
    q, k, v = qkv(cfg, (51, 52, 53))
    save("m64_n300", cfg, sparse.random_mask(cfg, 0.4, seed=3), q, k, v, seeds=(51, 52, 53))

    # full precision mode (ingest is the identity, core.py:188-193).
    cfg = core.AttnConfig(1, 1, 256, 64, precision="full")
    q, k, v = qkv(cfg, (61, 62, 63))
    save("full_prec", cfg, sparse.random_mask(cfg, 0.5, seed=9), q, k, v, seeds=(61, 62, 63))

    # --- mask builders -------------------------------------------------
    # avg-query pooling (masks.py:108-150); q scaled so scores spread out.
    cfg = core.AttnConfig(1, 2, 1024, 64, precision="bf16")
    q, k, v = qkv(cfg, (71, 72, 73), qmul=4.0)
    scores = masks.pooled_query_scores(q, k, cfg)
    tau = float(np.quantile(scores, 0.7))
    thr = masks.build_mask_avg_query(q, k, cfg, masks.MaskBuilderConfig("avg_query_threshold", tau=tau))
    topk = masks.build_mask_avg_query(q, k, cfg, masks.MaskBuilderConfig("avg_query_topk", top_k=100))
    fb = masks.build_mask_avg_query(q, k, cfg, masks.MaskBuilderConfig("avg_query_threshold", tau=1e9))
    save("avgq_thr", cfg, thr, q, k, v, seeds=(71, 72, 73), qmul=4.0, extra={
        "scores": scores, "tau": np.array(tau),
        "topk_padded": sparse.export_padded(topk).astype(np.int16), "top_k": np.array(100),
        "fallback_padded": sparse.export_padded(fb).astype(np.int16)})

    # top-k with heavy ties: bf16-rounded scores of a low-variance q.
    cfg = core.AttnConfig(1, 1, 512, 64, precision="bf16")
    q, k, v = qkv(cfg, (81, 82, 83), qmul=0.05)
    scores = masks.pooled_query_scores(q, k, cfg)
    topk = masks.build_mask_avg_query(q, k, cfg, masks.MaskBuilderConfig("avg_query_topk", top_k=37))
    save("avgq_topk_ties", cfg, topk, q, k, v, seeds=(81, 82, 83), qmul=0.05, outputs=False,
         extra={"scores": scores, "top_k": np.array(37),
                "n_unique_scores": np.array(len(np.unique(scores)))})

    # cached threshold from the full map (oracle.py:45-52, masks.py:94-105).
    cfg = core.AttnConfig(1, 2, 512, 64, precision="bf16")
    q, k, v = qkv(cfg, (91, 92, 93), qmul=3.0)
    amap = oracle.attention_map(q, k, cfg)
    tau = 4.0 / cfg.seq_len
    cm = masks.build_mask_cached(amap, cfg, tau)
    big = masks.build_mask_cached(amap, cfg, 2.0)  # tau > 1: argmax fallback only
    save("cached_thr", cfg, cm, q, k, v, seeds=(91, 92, 93), qmul=3.0, extra={
        "tau": np.array(tau), "map_sha": np.array(sha(amap.data)),
        "gmax": masks._group_max(core.analysis_scores(amap.data, cfg), cfg),
        "fallback_padded": sparse.export_padded(big).astype(np.int16)})


if __name__ == "__main__":
    main()
