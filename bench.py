#!/usr/bin/env python
"""FG-Attn layer benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2] [--density 0.45]

Workload (config "c2", BASELINE.json configs[1]): one Wan 2.1 1.3B attention
layer at 480p/81 frames -- B=1 per GPU, H=12, N=32760, D=128, M=128, bf16
Q/K/V ~ N(0,1) (synthetic), a uniform-random M x 1 slice mask keeping exactly
round(d*N) keys per query group (the random_mask count rule), d=0.45.

A step is one sparse_attention call over the whole layer with inputs
resident in HBM; L2 is flushed (512 MiB write) before every step, outside
the timed events.  ``value`` = algorithmic TFLOP/s = 4*D*sum(rows_g*count_g)
(perfmodel.py:104-105) / device time, summed over ranks.  Multi-GPU: one
process per GPU (torchrun), every rank runs its own batch element of the
layer (weak scaling, no collective on the hot path); NCCL is used only to
take the max time over ranks and to all-gather an output sample for the
bitwise cross-rank check.  ``--shard tiles`` instead splits ONE layer over the
ranks in contiguous work-balanced (head, group) tile ranges (strong scaling,
BASELINE configs c4/c5 "head-sharded"): value = the layer's FLOPs / the
slowest rank's time, and the ranks' outputs are NCCL-summed and checked
bitwise against a one-GPU run of the layer.

``e2e`` is the same metric through the public API from pinned HOST buffers
(``sparse_attention_host``): per step H2D of Q/K/V and the bit-packed slice
mask, K1b compaction, attention and D2H of O, overlapped over head slabs.  ``cpu_baseline`` (rank 0, N=1) times the oracle port of the
reference sparse_attention on the host cores on a bounded sample of the
same groups and doubles as the parity check of the GPU output.
``--impl reference`` times only that CPU path (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
METRIC = "FG-attn layer latency ms, TFLOP/s & speedup vs dense at Wan2.1 480p/720p"

CONFIGS = {
    # name: (heads, seq_len, head_dim, group_size, description)
    "c1": (2, 4096, 64, 128, "synthetic single-layer FG-attn, B=1, 2 heads, seq 4096, D=64"),
    "c2": (12, 32760, 128, 128, "Wan2.1-1.3B attention layer, 480p/81 frames: 12 heads, seq 32760, D=128"),
    "c3": (12, 75600, 128, 128, "Wan2.1-1.3B attention layer, 720p/81 frames: 12 heads, seq 75600, D=128"),
    "c4": (40, 32760, 128, 128, "Wan2.1-14B attention layer, 480p: 40 heads, seq 32760, D=128"),
    "c5": (40, 75600, 128, 128, "Wan2.1-14B attention layer, 720p: 40 heads, seq 75600, D=128"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--density", type=float, default=0.45)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--shard", default="batch", choices=["batch", "tiles"],
                    help="batch: every rank runs its own batch element (weak scaling, default); "
                         "tiles: one layer split over the ranks in contiguous work-balanced (head, group) "
                         "tile ranges (strong scaling, BASELINE configs c4/c5 head-sharded)")
    ap.add_argument("--no-extras", action="store_true", help="skip dense/e2e/cpu legs (for ncu)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-baseline work budget")
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


# ============================================================ CPU (oracle port) legs

def _cpu_pool_main(workdir: str):
    """Subprocess entry: OPENBLAS/OMP threads pinned to 1 before NumPy loads,
    one process per core, each computing whole groups with the oracle."""
    import multiprocessing as mp

    with open(os.path.join(workdir, "job.json")) as f:
        job = json.load(f)
    cores = job["cores"]
    ctx = mp.get_context("spawn")
    tasks = [(workdir, i) for i in range(len(job["groups"]))]
    with ctx.Pool(cores, initializer=_cpu_init, initargs=(workdir,)) as pool:
        pool.map(_cpu_noop, range(cores * 2))  # import + mmap warm-up outside the timing
        results = {}
        t0 = time.perf_counter()
        # all repetitions in one queue: the cores never idle at a per-repetition barrier
        for i, out in pool.imap_unordered(_cpu_task, tasks * job["reps"], chunksize=1):
            results[i] = out
        elapsed = time.perf_counter() - t0
    import numpy as np

    np.save(os.path.join(workdir, "out.npy"), np.stack([results[i] for i in range(len(tasks))]))
    with open(os.path.join(workdir, "timing.json"), "w") as f:
        json.dump({"seconds": elapsed, "reps": job["reps"]}, f)


_W = {}


def _cpu_init(workdir):
    import numpy as np

    sys.path.insert(0, ROOT)
    import oracle  # noqa: F401  (CPU-baseline leg: the only bench path that runs the oracle)

    with open(os.path.join(workdir, "job.json")) as f:
        _W["job"] = json.load(f)
    for name in ("q", "k", "v", "idx", "counts"):
        _W[name] = np.load(os.path.join(workdir, name + ".npy"), mmap_mode="r")
        float(np.asarray(_W[name]).sum())  # fault the pages in now, outside the timed region


def _cpu_noop(_):
    return 0


def _cpu_task(arg):
    import numpy as np
    import oracle

    _, i = arg
    job = _W["job"]
    g = job["groups"][i]
    m = job["group_size"]
    lo, hi = g * m, min(g * m + m, job["seq_len"])
    keys = np.asarray(_W["idx"][i, : int(_W["counts"][i])], dtype=np.int64)
    out = oracle.sparse_attention_group(np.asarray(_W["q"][lo:hi]), _W["k"], _W["v"], keys, job["scale"])
    full = np.zeros((m, _W["q"].shape[1]), np.float32)
    full[: hi - lo] = out
    return i, full


def run_cpu_baseline(qh, kh, vh, idx_rows, counts, groups, group_size, scale, cores, reps=1):
    """Time the oracle port on ``cores`` host processes.  Returns (seconds, outputs)."""
    import numpy as np

    workdir = tempfile.mkdtemp(prefix="fga_cpu_")
    np.save(os.path.join(workdir, "q.npy"), qh)
    np.save(os.path.join(workdir, "k.npy"), kh)
    np.save(os.path.join(workdir, "v.npy"), vh)
    np.save(os.path.join(workdir, "idx.npy"), idx_rows)
    np.save(os.path.join(workdir, "counts.npy"), counts)
    with open(os.path.join(workdir, "job.json"), "w") as f:
        json.dump({"groups": [int(g) for g in groups], "group_size": group_size, "seq_len": int(qh.shape[0]),
                   "scale": float(scale), "cores": cores, "reps": reps}, f)
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1",
               CUDA_VISIBLE_DEVICES="")
    subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-worker", workdir], check=True, env=env)
    with open(os.path.join(workdir, "timing.json")) as f:
        t = json.load(f)
    return t["seconds"], np.load(os.path.join(workdir, "out.npy"))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def reference_arm(args):
    """--impl reference: the oracle port of the reference sparse_attention on the
    host cores, same metric/config, rank 0 only."""
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, ROOT)
    import oracle

    heads, n, d, m, desc = CONFIGS[args.config]
    cores = host_cores()
    qh = oracle.bf16_round(oracle.gaussian((n, d), 1))
    kh = oracle.bf16_round(oracle.gaussian((n, d), 2))
    vh = oracle.bf16_round(oracle.gaussian((n, d), 3))
    g_count = -(-n // m)
    count = max(1, round(args.density * n))
    rng = np.random.Generator(np.random.Philox(args.seed))   # random_mask count rule (sparse.py:216-232)
    per_step = 4 * max(1, cores)  # four groups per core and step: per-task overheads amortised
    groups = [int(x) % g_count for x in range(per_step)]
    idx = np.stack([np.sort(rng.choice(n, size=count, replace=False)) for _ in groups]).astype(np.int32)
    counts = np.full(len(groups), count, np.int32)
    rows = np.array([min(m, n - g * m) for g in groups])
    flops_step = int(4 * d * (rows * count).sum())
    total = args.warmup + args.steps
    secs, _ = run_cpu_baseline(qh, kh, vh, idx, counts, groups, m, 1 / math.sqrt(d), cores, reps=total)
    per = secs / total
    value = flops_step / per / 1e12
    sample = (f"{per_step} query groups of head 0 per step ({count} keys each, {m} rows), "
              f"{total} steps timed together incl. {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": desc, "heads": heads, "seq_len": n, "head_dim": d, "group_size": m,
                   "density": args.density, "keys_per_group": count},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ============================================================ GPU helpers

class ClockSampler:
    """NVML polling (10 ms) of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x4: "sw_power_cap", 0x1: "gpu_idle",
               0x2: "applications_clocks_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


GATHER_CEILING_GBS = 12214.0  # L2 -> SMEM, random 2*D-byte rows (profiles/r01/gather_bench2.log)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, density):
    """Per-launch dram bytes of the attention kernel from the committed ncu capture, if it matches."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(f"{config}@{density}")
        return None if e is None else e["dram_bytes_per_launch"]
    except Exception:
        return None


def timed_steps(torch, fn, steps, flush, stream):
    """Per-step CUDA-event times (ms) on ``stream``; L2 flushed before each step, untimed."""
    ts = []
    for _ in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ts]


# ============================================================ our arm

def ours(args):
    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    sys.path.insert(0, ROOT)
    import paper_2509_16518_b200 as fga
    from paper_2509_16518_b200 import _lib

    lib = _lib.load()
    heads, n, d, m, desc = CONFIGS[args.config]
    cfg = fga.AttnConfig(1, heads, n, d, group_size=m, precision="bf16")
    stream = torch.cuda.current_stream()
    gen = torch.Generator(device=dev).manual_seed(1234 + args.seed)   # identical on every rank (bitwise check)
    q = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    k = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    v = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    count = max(1, round(args.density * n))
    rows_g = cfg.batch * cfg.heads * cfg.num_groups
    keep = torch.empty((1, heads, cfg.num_groups, n), dtype=torch.uint8, device=dev)
    _lib.call("fga_random_keep", rows_g, n, count, 77 + args.seed, keep.data_ptr(), stream.cuda_stream)
    mask = fga.compact_keep(keep, m)
    rep = fga.count_flops(cfg, mask)
    flops = rep.flops_matmul           # 4*D*pairs: the roofline numerator (softmax excluded)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    strong = args.shard == "tiles"
    if strong:
        from paper_2509_16518_b200 import shard

        ranges = shard.partition_tiles(shard.tile_work(cfg, mask.counts.cpu().numpy()), world)
        my_range = ranges[rank]
        out_buf = torch.zeros(cfg.dims, dtype=torch.bfloat16, device=dev)

        def step():
            return shard.sparse_attention_shard(q, k, v, mask, cfg, my_range, out_buf)
    else:
        def step():
            return fga.sparse_attention(q, k, v, mask, cfg)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        times = timed_steps(torch, step, args.steps, flush, stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    wall = time.perf_counter() - wall0
    kernel_ms = sum(times) / len(times)
    if dist:
        t = torch.tensor([kernel_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kernel_ms = float(t.item())
    out = step()
    torch.cuda.synchronize()

    peak, peak_sus, hbm_peak, peak_src = measured_peaks()
    achieved = flops / (kernel_ms * 1e-3) / 1e12  # strong: the whole layer's FLOPs in the slowest rank's time
    gathered = int(rep.density * cfg.batch * heads * cfg.num_groups * n) * 4 * d  # K + V rows, bf16
    value = achieved if strong else achieved * world
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": kernel_ms, "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (N(0,1) bf16 Q/K/V, uniform random slice mask)",
        "config": {"workload": desc, "config": args.config, "batch_per_gpu": 1 if not strong else None,
                   "global_batch": 1 if strong else world,
                   "heads": heads, "seq_len": n, "head_dim": d, "group_size": m, "density": args.density,
                   "keys_per_group": count,
                   "parallelism": (f"tiles{world} (one layer, work-balanced (head, group) tile ranges, strong)" if strong
                                   else f"dp{world} (batch-sharded, weak)"),
                   "l2": "flushed between steps (512 MiB write, untimed)"},
        "latency_ms": kernel_ms,
        "gpu_launches": args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus if peak_sus else None,
                     "peak_source": peak_src, "traffic": ncu_traffic(args.config, args.density),
                     "algorithmic_flops_per_launch": flops,
                     "gathered_kv_bytes_per_launch": gathered,
                     "kernel": "fga_attn_ws_kernel",
                     # the gathered K/V rows move L2 -> SMEM; their ceiling is the measured random-row
                     # gather rate (scripts/gather_bench2.cu, profiles/r01/gather_bench2.log)
                     "gather": {"achieved_gbs": gathered / (kernel_ms * 1e-3) / 1e9, "ceiling_gbs": GATHER_CEILING_GBS,
                                "frac": gathered / (kernel_ms * 1e-3) / 1e9 / GATHER_CEILING_GBS,
                                "ceiling_source": "measured: cp.async warp-per-chunk gather of random 256-byte rows"}},
        "clocks": clk.summary(),
        "wall_s_timed_region": wall,
    }

    # ---- validation (NCCL, outside the timed region)
    if strong:
        # the ranks' tile ranges, summed over ranks (zeros elsewhere), must equal the one-GPU layer bitwise
        full = fga.sparse_attention(q, k, v, mask, cfg)
        red = out_buf.clone()
        if dist:
            dist.all_reduce(red)
        line["reassembled_bitwise_equal"] = bool(torch.equal(red, full))
        line["tile_ranges"] = ranges
        out = full
    elif dist:
        from paper_2509_16518_b200.shard import gather_outputs

        sample = out[0, 0, :256].contiguous()
        allo = gather_outputs(sample)
        line["cross_rank_bitwise_equal"] = bool(all(torch.equal(allo[0], allo[r]) for r in range(world)))

    if not args.no_extras:
        e2e = e2e_leg(args, torch, fga, cfg, q, k, v, keep, out, flops, flush, stream, world, dist, strong)
        if rank == 0:
            line["e2e"] = e2e
    if not args.no_extras and rank == 0:
        extras(args, torch, np, fga, _lib, cfg, q, k, v, keep, mask, out, flops, flush, stream, line, world,
               hbm_peak, peak_src, count)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def e2e_leg(args, torch, fga, cfg, q, k, v, keep, out, flops, flush, stream, world, dist, strong):
    """The metric end to end through the public API from pinned HOST buffers, on every rank at
    once (each rank its own batch element; max time over ranks): per step H2D of Q/K/V and the
    bit-packed slice mask, K1b compaction, attention and D2H of O, overlapped over head slabs."""
    bits = fga.pack_keep_bits(keep)
    hq, hk, hv = (x.cpu().pin_memory() for x in (q, k, v))
    hbits = bits.cpu().pin_memory()
    hout = torch.empty(cfg.dims, dtype=torch.bfloat16).pin_memory()

    def e2e_step():
        fga.sparse_attention_host(hq, hk, hv, hbits, cfg, out=hout)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t_e = timed_steps(torch, e2e_step, max(3, args.steps // 2), flush, stream)
    e_ms = sum(t_e) / len(t_e)
    if dist:
        t = torch.tensor([e_ms], device=q.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = 3 * q.numel() * 2 + bits.numel() * 4
    e2e_err = float((hout.float() - out.float().cpu()).abs().max())
    # strong (--shard tiles): every rank runs the whole layer from its host buffers, so the
    # layer rate is one layer per (slowest) step, not world layers
    layers = 1 if strong else world
    return {"value": flops / (e_ms * 1e-3) / 1e12 * layers, "unit": "TFLOP/s", "ms_per_step": e_ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": out.numel() * 2, "ranks": world,
            "path": "sparse_attention_host: pinned host Q/K/V + bit-packed slice mask -> H2D | "
                    "fga_compact_bits + fga_sparse_attn_fwd | D2H, overlapped over 5 head slabs (the last one a "
                    "single head, its query groups in 2 runs); every rank at once, max time over ranks",
            "max_abs_diff_vs_device_path": e2e_err}


def extras(args, torch, np, fga, _lib, cfg, q, k, v, keep, mask, out, flops, flush, stream, line, world,
           hbm_peak, peak_src, count):
    heads, n, d, m = cfg.heads, cfg.seq_len, cfg.head_dim, cfg.group_size
    kernel_ms = line["ms_per_step"]
    # ---- dense denominators on the same GPU: our dense kernel + torch SDPA backends
    dense = {}
    t_own = timed_steps(torch, lambda: fga.flash_attention(q, k, v, cfg), max(3, args.steps // 2), flush, stream)
    dense["own_tcgen05_ms"] = sorted(t_own)[len(t_own) // 2]
    from torch.nn.attention import SDPBackend, sdpa_kernel

    for name, be in (("sdpa_cudnn_ms", SDPBackend.CUDNN_ATTENTION), ("sdpa_flash_ms", SDPBackend.FLASH_ATTENTION),
                     ("sdpa_efficient_ms", SDPBackend.EFFICIENT_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                torch.nn.functional.scaled_dot_product_attention(q, k, v)
                tt = timed_steps(torch, lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v),
                                 max(3, args.steps // 2), flush, stream)
            dense[name] = sorted(tt)[len(tt) // 2]
        except Exception as e:  # backend not available for this shape
            dense[name] = None
    best = min(x for x in dense.values() if x)
    dense["best_ms"] = best
    dense["dense_flops"] = 4 * d * heads * n * n
    line["dense"] = dense
    line["speedup_vs_dense"] = best / kernel_ms

    # ---- K1b compaction (HBM-bound): keep bytes (or bits) read + 4*count written (+ counts)
    live = 4 * int(mask.counts.sum().item()) + 4 * mask.counts.numel()
    t_c = timed_steps(torch, lambda: fga.compact_keep(keep, m), max(3, args.steps), flush, stream)
    c_ms = sorted(t_c)[len(t_c) // 2]
    c_bytes = keep.numel() + live
    bits_dev = fga.pack_keep_bits(keep)
    t_b = timed_steps(torch, lambda: fga.compact_keep_bits(bits_dev, m, n), max(3, args.steps), flush, stream)
    b_ms = sorted(t_b)[len(t_b) // 2]
    b_bytes = bits_dev.numel() * 4 + live
    line["mask_build"] = {"kernel": "fga_compact_kernel", "ms": c_ms, "bytes": c_bytes,
                          "achieved_gbs": c_bytes / (c_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                          "frac": c_bytes / (c_ms * 1e-3) / 1e9 / hbm_peak, "peak_source": peak_src,
                          "bits_kernel": "fga_compact_bits_kernel", "bits_ms": b_ms, "bits_bytes": b_bytes,
                          "bits_achieved_gbs": b_bytes / (b_ms * 1e-3) / 1e9,
                          "bits_frac": b_bytes / (b_ms * 1e-3) / 1e9 / hbm_peak,
                          "layer_ms_incl_compaction": kernel_ms + min(c_ms, b_ms)}

    # ---- K1a threshold builders on the same Q/K (masks.py:94-150), each to a device mask:
    #      the cached-threshold builder on the tensor cores (the paper recalibrates it every 15
    #      denoising iterations) and the avg-query builders
    from paper_2509_16518_b200 import masks as fmasks

    builders = {}
    for name, fn in (
            ("cached_threshold_ms", lambda: fmasks.build_mask_cached_qk(q, k, cfg, 0.5 / n, device_result=True)),
            ("avg_query_topk_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
                "avg_query_topk", top_k=count), device_result=True)),
            ("avg_query_threshold_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
                "avg_query_threshold", tau=1.0 / d), device_result=True))):
        tb = timed_steps(torch, fn, 3, flush, stream)
        builders[name] = sorted(tb)[len(tb) // 2]
    builders["cached_amortised_per_iteration_ms"] = builders["cached_threshold_ms"] / 15
    line["mask_builders"] = builders

    # ---- CPU baseline (oracle port, rank 0, N=1 only) + parity of the same groups
    if world == 1:
        cores = host_cores()
        per_group_s = 4 * d * m * count / 25e9      # ~25 GFLOP/s per core for the NumPy port
        budget = max(cores, int(args.cpu_seconds * cores / per_group_s))
        units = [(h, g) for h in range(heads) for g in range(cfg.num_groups)][:budget]
        heads_used = sorted({h for h, _ in units})
        res_err, cpu_secs, f_sample = 0.0, 0.0, 0
        for h in heads_used:   # one worker pool run per head (K/V of that head mmap-shared)
            groups = [g for hh, g in units if hh == h]
            qh, kh, vh = (x[0, h].float().cpu().numpy() for x in (q, k, v))
            idx_rows = mask.idx[0, h, groups].cpu().numpy()
            cnts = mask.counts[0, h, groups].cpu().numpy()
            secs, cpu_out = run_cpu_baseline(qh, kh, vh, idx_rows, cnts, groups, m, cfg.scale, cores)
            cpu_secs += secs
            rows = np.array([min(m, n - g * m) for g in groups])
            f_sample += int(4 * d * (rows * cnts.astype(np.int64)).sum())
            gpu_rows = out[0, h].float().cpu().numpy()
            for j, g in enumerate(groups):
                lo, hi = g * m, min(g * m + m, n)
                res_err = max(res_err, float(np.abs(gpu_rows[lo:hi] - cpu_out[j, : hi - lo]).max()))
        cpu_val = f_sample / cpu_secs / 1e12
        full = len(units) == heads * cfg.num_groups
        line["cpu_baseline"] = {"value": cpu_val, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                                "sample": (f"{'the whole layer' if full else 'a bounded sample'}: {len(units)} query "
                                           f"groups x {count} keys over {len(heads_used)} heads, "
                                           "oracle.sparse_attention_group, one process per core"),
                                "seconds": cpu_secs, "core_seconds": cpu_secs * cores,
                                "gpu_vs_cpu_ratio": line["value"] / cpu_val}
        line["parity"] = {"max_abs_err_vs_oracle": res_err, "tolerance": 2e-2, "groups_checked": len(units),
                          "output_dtype": "bf16"}


def main():
    args = parse()
    if args.cpu_worker:
        _cpu_pool_main(args.cpu_worker)
        return
    if args.impl == "reference":
        reference_arm(args)
        return
    ours(args)


if __name__ == "__main__":
    main()
