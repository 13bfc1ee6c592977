#!/usr/bin/env python
"""FG-Attn layer benchmark (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cX]
                    [--density 0.45] [--shard heads|tiles|batch] [--dry-run]

Workloads (BASELINE.json configs): synthetic bf16 Q/K/V ~ N(0,1) of a Wan 2.1 attention layer,
B=1, D=128, M=128 (G = ceil(N/M) query groups), and a uniform-random M x 1 slice mask keeping
exactly round(d*N) keys per group (the random_mask count rule, sparse.py:216-232), d=0.45.

* N=1 (default): config c2 = Wan 2.1 1.3B at 480p (H=12, N=32760), BASELINE.json configs[1].
* N>1: config c4 = Wan 2.1 14B at 480p (H=40, N=32760) head-sharded over the N GPUs (strong
  scaling: contiguous head blocks, BASELINE.json configs[3]); at N=8 also c5 (14B at 720p,
  N=75600) with the 10-90% density sweep (configs[4]).  ``--shard tiles`` splits a layer whose
  heads do not divide evenly into work-balanced (head, group) tile ranges; ``--shard batch`` runs
  one layer per GPU (weak scaling).  No collective runs on the hot path; NCCL only takes the max
  time over ranks and gathers the outputs once, outside the timed region, for the bitwise check
  against a one-GPU run of the whole layer.

``python bench.py --gpus N`` without torchrun re-launches itself under
``torch.distributed.run`` with N processes (one per GPU); under torchrun, WORLD_SIZE must equal
``--gpus``.

A step is one sparse_attention call over the (shard of the) layer with inputs resident in HBM;
L2 is flushed (512 MiB write) before every step, outside the timed events.  ``value`` =
algorithmic TFLOP/s = 4*D*sum(rows_g*count_g) (perfmodel.py:104-105) of the whole layer / the
slowest rank's device time.  ``e2e`` is the same metric through the public API from pinned HOST
buffers (``sparse_attention_host``: H2D of Q/K/V and the bit-packed slice mask, K1b compaction,
attention, D2H of O), every rank at once, max over ranks.  ``parity`` recomputes >= 2 whole heads
with the CPU oracle; at N=1 that leg is also timed as ``cpu_baseline``.

``--impl reference`` (the reference arm) times the UNMODIFIED reference package
(``baseline/_ref/sliceattn``: ``sliceattn.sparse.sparse_attention`` through its public API, with
the reference's own ``new_tensor`` / ``random_mask``) on the host cores, one single-head call per
task, one process per core, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
SWEEP = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 on one GPU, c4 head-sharded on several")
    ap.add_argument("--density", type=float, default=0.45)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--shard", default=None, choices=["heads", "tiles", "batch"],
                    help="N>1: heads (default when the heads divide evenly), tiles (work-balanced (head, "
                         "group) ranges of one layer), batch (one layer per GPU, weak scaling)")
    ap.add_argument("--sweep", default=None, choices=["on", "off"],
                    help="c5 density sweep 10-90%% (default: on at 8 GPUs)")
    ap.add_argument("--no-extras", action="store_true", help="skip dense/e2e/parity/builder legs (for ncu)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU-baseline work budget")
    ap.add_argument("--ref-seconds", type=float, default=150.0, help="reference-arm work budget")
    ap.add_argument("--dry-run", action="store_true",
                    help="host logic only (CPU, gloo): launch, partition, collectives; no kernels")
    ap.add_argument("--allow-shared-gpu", action="store_true",
                    help="let several ranks share a GPU (gloo for the validation collectives)")
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--ref-worker", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


def default_config(args, world):
    return args.config or ("c2" if world == 1 else "c4")


def default_shard(args, world, heads):
    if args.shard:
        return args.shard
    if world == 1:
        return "heads"
    return "heads" if heads % world == 0 else "tiles"


# ============================================================ self-launch

def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args) -> int:
    """``--gpus N`` outside torchrun: run this script under torch.distributed.run, N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))).returncode


# ============================================================ CPU legs (oracle port / reference)

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
        for i, out in pool.imap_unordered(_cpu_task, tasks, chunksize=1):
            results[i] = out
        elapsed = time.perf_counter() - t0
    import numpy as np

    np.save(os.path.join(workdir, "out.npy"), np.stack([results[i] for i in range(len(tasks))]))
    with open(os.path.join(workdir, "timing.json"), "w") as f:
        json.dump({"seconds": elapsed}, f)


_W = {}


def _cpu_init(workdir):
    import numpy as np

    sys.path.insert(0, ROOT)
    import oracle  # noqa: F401  (parity / cpu_baseline leg: the oracle as the checker)

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
    h, g = job["groups"][i]
    m = job["group_size"]
    lo, hi = g * m, min(g * m + m, job["seq_len"])
    keys = np.asarray(_W["idx"][i, : int(_W["counts"][i])], dtype=np.int64)
    out = oracle.sparse_attention_group(np.asarray(_W["q"][h, lo:hi]), _W["k"][h], _W["v"][h], keys, job["scale"])
    full = np.zeros((m, _W["q"].shape[-1]), np.float32)
    full[: hi - lo] = out
    return i, full


def run_cpu_units(qh, kh, vh, idx_rows, counts, units, group_size, scale, cores):
    """Oracle port on ``cores`` host processes over (head, group) units; qh/kh/vh [H', N, D].
    Returns (seconds, outputs [len(units), M, D])."""
    import numpy as np

    workdir = tempfile.mkdtemp(prefix="fga_cpu_")
    for name, arr in (("q", qh), ("k", kh), ("v", vh), ("idx", idx_rows), ("counts", counts)):
        np.save(os.path.join(workdir, name + ".npy"), arr)
    with open(os.path.join(workdir, "job.json"), "w") as f:
        json.dump({"groups": [[int(h), int(g)] for h, g in units], "group_size": group_size,
                   "seq_len": int(qh.shape[1]), "scale": float(scale), "cores": cores}, f)
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


def _ref_head_inputs(sa, job, h):
    """The reference's own generators for head h (core.py:150-175, sparse.py:216-232)."""
    cfg = sa.core.AttnConfig(1, 1, job["seq_len"], job["head_dim"], group_size=job["group_size"],
                             precision="bf16")
    q = sa.core.new_tensor(cfg, "gaussian", seed=1000 + h)
    k = sa.core.new_tensor(cfg, "gaussian", seed=2000 + h)
    v = sa.core.new_tensor(cfg, "gaussian", seed=3000 + h)
    mask = sa.sparse.random_mask(cfg, job["density"], seed=h)
    return cfg, q, k, v, mask


def _ref_worker_main(workdir: str):
    """Reference arm subprocess: one process per core, each runs its share of the single-head
    sparse_attention calls of the job, the inputs of its heads built (untimed) first."""
    import multiprocessing as mp

    with open(os.path.join(workdir, "job.json")) as f:
        job = json.load(f)
    cores = job["cores"]
    ctx = mp.get_context("spawn")
    start = ctx.Barrier(cores + 1)
    q_out = ctx.Queue()
    procs = [ctx.Process(target=_ref_proc, args=(workdir, w, start, q_out)) for w in range(cores)]
    for p in procs:
        p.start()
    start.wait()   # every worker has built its inputs and run its warm-up call
    res = [q_out.get() for _ in procs]
    for p in procs:
        p.join()
    t0 = min(r["t0"] for r in res)
    t1 = max(r["t1"] for r in res)
    with open(os.path.join(workdir, "timing.json"), "w") as f:
        json.dump({"seconds": t1 - t0, "tasks": sum(r["tasks"] for r in res),
                   "flops": sum(r["flops"] for r in res), "warm_task_s": [r["warm_s"] for r in res]}, f)


def _ref_proc(workdir, w, start, q_out):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import numpy as np  # noqa: F401
    import sliceattn.core
    import sliceattn.sparse
    import sliceattn as sa

    with open(os.path.join(workdir, "job.json")) as f:
        job = json.load(f)
    mine = [h for t, h in enumerate(job["tasks"]) if t % job["cores"] == w]
    inputs = {h: _ref_head_inputs(sa, job, h) for h in sorted(set(mine))}
    warm_s = 0.0
    if mine:
        t = time.perf_counter()
        sa.sparse.sparse_attention(*inputs[mine[0]][1:], inputs[mine[0]][0])   # warm-up call
        warm_s = time.perf_counter() - t
    start.wait()
    t0 = time.perf_counter()
    flops = 0
    for h in mine:
        cfg, q, k, v, mask = inputs[h]
        sa.sparse.sparse_attention(q, k, v, mask, cfg)
        for g in range(cfg.num_groups):
            lo, hi = cfg.group_bounds(g)
            flops += 4 * cfg.head_dim * (hi - lo) * mask.keys_for(0, 0, g).size
    t1 = time.perf_counter()
    q_out.put({"t0": t0, "t1": t1, "tasks": len(mine), "flops": flops, "warm_s": warm_s})


def reference_arm(args):
    """--impl reference: the unmodified reference sparse_attention (baseline/_ref) on the host
    cores, same metric / config / density; rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    cfg_name = default_config(args, world)
    heads, n, d, m, desc = CONFIGS[cfg_name]
    cores = host_cores()
    ref_dir = os.path.join(ROOT, "baseline", "_ref", "sliceattn")
    line = {"impl": "reference", "metric": METRIC, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True}
    if not os.path.isdir(ref_dir):
        line.update({"unavailable": "baseline/_ref/sliceattn missing (pip install --target baseline/_ref failed)"})
        print(json.dumps(line), flush=True)
        return
    # per-head single-core time at this config ~ 4*D*rows*count*G / 30 GFLOP/s (survey: 37.8 at c2)
    count = max(1, round(args.density * n))
    g_count = -(-n // m)
    head_flops = 4 * d * n * count
    est_task_s = head_flops / 30e9
    per_step = max(1, min(heads, cores, int(args.ref_seconds * cores / max(1, args.steps) / est_task_s)))
    tasks = [(s * per_step + i) % heads for s in range(args.steps) for i in range(per_step)]
    workdir = tempfile.mkdtemp(prefix="fga_ref_")
    job = {"tasks": tasks, "cores": min(cores, len(tasks)), "seq_len": n, "head_dim": d, "group_size": m,
           "density": args.density}
    with open(os.path.join(workdir, "job.json"), "w") as f:
        json.dump(job, f)
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1",
               CUDA_VISIBLE_DEVICES="")
    subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-worker", workdir], check=True, env=env)
    with open(os.path.join(workdir, "timing.json")) as f:
        t = json.load(f)
    value = t["flops"] / t["seconds"] / 1e12
    per = t["seconds"] / args.steps
    sample = (f"{per_step} of the layer's {heads} heads per step ({args.steps} steps, {len(tasks)} single-head "
              f"sliceattn.sparse.sparse_attention calls of {g_count} groups x {count} keys, precision='bf16'), "
              f"{job['cores']} processes, one per core, OPENBLAS_NUM_THREADS=1; inputs from the reference's "
              f"new_tensor/random_mask, built untimed; one untimed warm-up call per process")
    line.update({
        "value": value, "ms_per_step": per * 1e3, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference new_tensor gaussian, random_mask)",
        "config": {"workload": desc, "config": cfg_name, "heads": heads, "seq_len": n, "head_dim": d,
                   "group_size": m, "density": args.density, "keys_per_group": count},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": job["cores"], "kind": "reference",
                         "sample": sample, "seconds": t["seconds"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_path": "baseline/_ref/sliceattn/sparse.py:111-156 (pip install --no-index --target baseline/_ref "
                          "of /root/reference/pkg, unmodified)",
    })
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


class Dist:
    """torch.distributed plumbing: NCCL, or gloo when ranks share a GPU / in a dry run."""

    def __init__(self, world, rank, local, dev, backend):
        self.world, self.rank, self.local, self.dev, self.backend = world, rank, local, dev, backend
        self.d = None
        if world > 1:
            import torch.distributed as dist

            if backend == "nccl":
                dist.init_process_group("nccl", device_id=dev)
            else:
                dist.init_process_group("gloo")
            self.d = dist

    def barrier(self):
        if self.d:
            self.d.barrier()

    def max(self, x: float) -> float:
        if not self.d:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device=self.dev if self.backend == "nccl" else "cpu")
        self.d.all_reduce(t, op=self.d.ReduceOp.MAX)
        return float(t.item())

    def gather(self, t):
        """All-gather equally shaped tensors -> [world, ...] (on rank-local device memory)."""
        import torch

        if not self.d:
            return t[None]
        if self.backend == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.d.all_gather_into_tensor(out, t.contiguous())
            return out
        parts = [torch.empty_like(t, device="cpu") for _ in range(self.world)]
        self.d.all_gather(parts, t.cpu().contiguous())
        return torch.stack(parts).to(t.device)

    def close(self):
        if self.d:
            self.d.destroy_process_group()


# ============================================================ our arm

def env_world():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def dry_run(args):
    """Host logic without kernels (CPU box): the launch, the partition and the collectives the
    GPU run uses, over gloo."""
    import torch

    world, rank, local = env_world()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    sys.path.insert(0, ROOT)
    from paper_2509_16518_b200 import shard
    from paper_2509_16518_b200.core import AttnConfig

    cfg_name = default_config(args, world)
    heads, n, d, m, desc = CONFIGS[cfg_name]
    mode = default_shard(args, world, heads)
    dist = Dist(world, rank, local, torch.device("cpu"), "gloo")
    cfg = AttnConfig(1, heads, n, d, group_size=m, precision="bf16")
    count = max(1, round(args.density * n))
    line = {"dry_run": True, "n_gpus": world, "config": {"workload": desc, "config": cfg_name}, "shard": mode}
    if mode == "heads":
        blocks = shard.head_blocks(heads, world)
        h0, h1 = blocks[rank]
        mine = torch.full((h1 - h0,), float(rank))
        allv = dist.gather(mine)
        line["head_blocks"] = blocks
        line["gather_ok"] = bool(all((allv[r] == r).all() for r in range(world)))
    else:
        import numpy as np

        work = shard.tile_work(cfg, np.full(cfg.batch * heads * cfg.num_groups, count))
        ranges = shard.partition_tiles(work, world)
        line["tile_ranges"] = ranges
        allr = dist.gather(torch.tensor(ranges[rank]))
        line["gather_ok"] = [tuple(int(x) for x in r) for r in allr] == [tuple(r) for r in ranges]
    line["max_rank_allreduce"] = dist.max(float(rank))  # the max-over-ranks reduction the timing uses
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


def make_layer(torch, fga, _lib, cfg, density, seed, dev):
    """Synthetic layer, identical on every rank: bf16 Q/K/V ~ N(0,1) and exact-count keep bytes."""
    gen = torch.Generator(device=dev).manual_seed(1234 + seed)
    q = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    k = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    v = torch.randn(cfg.dims, device=dev, dtype=torch.float32, generator=gen).to(torch.bfloat16)
    keep = make_keep(torch, _lib, cfg, density, seed, dev)
    return q, k, v, keep


def make_keep(torch, _lib, cfg, density, seed, dev):
    count = max(1, round(density * cfg.seq_len))
    rows = cfg.batch * cfg.heads * cfg.num_groups
    keep = torch.empty((cfg.batch, cfg.heads, cfg.num_groups, cfg.seq_len), dtype=torch.uint8, device=dev)
    _lib.call("fga_random_keep", rows, cfg.seq_len, count, 77 + seed, keep.data_ptr(),
              torch.cuda.current_stream(dev).cuda_stream)
    return keep


def ours(args):
    import numpy as np
    import torch

    world, rank, local = env_world()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus} (run without torchrun to self-launch)")
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device (use --dry-run for the host logic)")
    shared = world > ndev
    if shared and not args.allow_shared_gpu:
        raise SystemExit(f"bench.py: {world} ranks but {ndev} GPU(s); pass --allow-shared-gpu to share them")
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    dist = Dist(world, rank, local, dev, "gloo" if shared else "nccl")

    sys.path.insert(0, ROOT)
    import paper_2509_16518_b200 as fga
    from paper_2509_16518_b200 import _lib, shard

    _lib.load()
    cfg_name = default_config(args, world)
    heads, n, d, m, desc = CONFIGS[cfg_name]
    mode = default_shard(args, world, heads)
    if mode == "heads" and heads % world:
        raise SystemExit(f"bench.py: {heads} heads do not split over {world} GPUs; use --shard tiles")
    cfg = fga.AttnConfig(1, heads, n, d, group_size=m, precision="bf16")
    stream = torch.cuda.current_stream()
    q, k, v, keep = make_layer(torch, fga, _lib, cfg, args.density, args.seed, dev)
    count = max(1, round(args.density * n))
    mask = fga.compact_keep(keep, m)
    mask.validated = True  # exactly `count` distinct keys per row (fga_random_keep)
    layer_flops = fga.count_flops(cfg, mask).flops_matmul  # 4*D*pairs: the roofline numerator
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # ---- this rank's share of the work
    if mode == "heads":
        h0, h1 = shard.head_blocks(heads, world)[rank]
        if world == 1:
            lcfg, lq, lk, lv, lkeep, lmask = cfg, q, k, v, keep, mask
        else:
            lcfg = fga.AttnConfig(1, h1 - h0, n, d, group_size=m, precision="bf16")
            lq, lk, lv = (x[:, h0:h1].contiguous() for x in (q, k, v))
            lkeep = keep[:, h0:h1].contiguous()
            lmask = fga.compact_keep(lkeep, m)
            lmask.validated = True

        def step():
            return fga.sparse_attention(lq, lk, lv, lmask, lcfg)
        rank_flops = fga.count_flops(lcfg, lmask).flops_matmul
        layers_per_step = 1
    elif mode == "tiles":
        ranges = shard.partition_tiles(shard.tile_work(cfg, mask.counts.cpu().numpy()), world)
        my_range = ranges[rank]
        out_buf = torch.zeros(cfg.dims, dtype=torch.bfloat16, device=dev)
        lcfg, lq, lk, lv, lkeep, lmask = cfg, q, k, v, keep, mask

        def step():
            return shard.sparse_attention_shard(q, k, v, mask, cfg, my_range, out_buf)
        rank_flops = None
        layers_per_step = 1
    else:  # batch: every rank runs the whole layer (its own batch element), weak scaling
        lcfg, lq, lk, lv, lkeep, lmask = cfg, q, k, v, keep, mask

        def step():
            return fga.sparse_attention(q, k, v, mask, cfg)
        rank_flops = layer_flops
        layers_per_step = world

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(dev_index) as clk:
        times = timed_steps(torch, step, args.steps, flush, stream)
    torch.cuda.synchronize()
    dist.barrier()
    wall = time.perf_counter() - wall0
    my_ms = sum(times) / len(times)
    kernel_ms = dist.max(my_ms)
    out = step()
    torch.cuda.synchronize()

    peak, peak_sus, hbm_peak, peak_src = measured_peaks()
    value = layer_flops * layers_per_step / (kernel_ms * 1e-3) / 1e12
    # roofline of the kernel on this GPU: its own FLOPs in its own time (rank 0)
    k_flops = rank_flops if rank_flops is not None else layer_flops / world
    achieved = k_flops / (my_ms * 1e-3) / 1e12
    # gathered K+V rows (2 x 2D bytes per listed key and 128-row tile; one tile per group at M=128)
    tiles_per_group = -(-m // 128)
    gathered = int(lmask.counts.sum().item()) * 4 * d * tiles_per_group
    if mode == "tiles":
        gathered //= world
    parallelism = {"heads": f"heads{world} (contiguous head blocks of one layer, strong)",
                   "tiles": f"tiles{world} (one layer, work-balanced (head, group) tile ranges, strong)",
                   "batch": f"dp{world} (one layer per GPU, weak)"}[mode]
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": kernel_ms, "higher_is_better": True,
        "scaling": "weak" if mode == "batch" else "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (N(0,1) bf16 Q/K/V, uniform random slice mask)",
        "config": {"workload": desc, "config": cfg_name, "global_batch": layers_per_step if mode == "batch" else 1,
                   "heads": heads, "seq_len": n, "head_dim": d, "group_size": m, "density": args.density,
                   "keys_per_group": count, "parallelism": parallelism,
                   "heads_per_gpu": lcfg.heads if mode == "heads" else None,
                   "l2": "flushed between steps (512 MiB write, untimed)"},
        "latency_ms": kernel_ms,
        "gpu_launches": args.steps,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "frac_of_sustained": achieved / peak_sus if peak_sus else None,
                     "peak_source": peak_src, "traffic": ncu_traffic(cfg_name, args.density) if world == 1 else None,
                     "algorithmic_flops_per_launch": k_flops, "gathered_kv_bytes_per_launch": gathered,
                     "kernel": "fga_attn_ws_kernel",
                     "gather": {"achieved_gbs": gathered / (my_ms * 1e-3) / 1e9, "ceiling_gbs": GATHER_CEILING_GBS,
                                "frac": gathered / (my_ms * 1e-3) / 1e9 / GATHER_CEILING_GBS,
                                "ceiling_source": "measured: cp.async warp-per-chunk gather of random 256-byte rows"}},
        "clocks": clk.summary(),
        "wall_s_timed_region": wall,
    }
    if shared:
        line["shared_gpu"] = f"{world} ranks on {ndev} GPU(s): times include contention (validation run)"

    # ---- validation (outside the timed region): outputs vs a one-GPU run of the whole layer
    if world > 1:
        if mode == "heads":
            allo = dist.gather(out)                      # [world, 1, H/world, N, D]
            if rank == 0:
                full = fga.sparse_attention(q, k, v, mask, cfg)
                re = torch.cat([allo[r] for r in range(world)], dim=1)
                line["reassembled_bitwise_equal"] = bool(torch.equal(re, full))
                line["head_blocks"] = shard.head_blocks(heads, world)
                t1 = timed_steps(torch, lambda: fga.sparse_attention(q, k, v, mask, cfg), 5, flush, stream)
                line["layer_one_gpu_ms"] = sorted(t1)[len(t1) // 2]
                out = full
        elif mode == "tiles":
            red = dist.gather(out_buf).float().sum(0).to(torch.bfloat16)
            if rank == 0:
                full = fga.sparse_attention(q, k, v, mask, cfg)
                line["reassembled_bitwise_equal"] = bool(torch.equal(red, full))
                line["tile_ranges"] = ranges
                out = full
        else:
            allo = dist.gather(out[0, 0, :256].contiguous())
            line["cross_rank_bitwise_equal"] = bool(all(torch.equal(allo[0], allo[r]) for r in range(world)))
    elif mode == "tiles":
        out = fga.sparse_attention(q, k, v, mask, cfg)

    if not args.no_extras:
        e2e = e2e_leg(args, torch, fga, lcfg, lq, lk, lv, lkeep, layer_flops * layers_per_step, flush, stream, dist,
                      mode, out if mode != "heads" or world == 1 else None)
        if rank == 0:
            line["e2e"] = e2e
        if rank == 0:
            try:  # rank-0-only legs (no collectives): a failure there must not lose the contract line
                extras(args, torch, np, fga, lcfg, lq, lk, lv, lkeep, lmask, out if world == 1 else None, my_ms,
                       flush, stream, line, world, hbm_peak, peak_src, count)
            except Exception as exc:  # noqa: BLE001
                line["extras_error"] = f"{type(exc).__name__}: {exc}"
        sweep = args.sweep == "on" or (args.sweep is None and world == 8 and mode == "heads")
        if sweep:
            res = c5_sweep(args, torch, fga, _lib, shard, dist, dev, flush, stream, world, rank)
            if rank == 0:
                line["c5_sweep"] = res
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()


def e2e_leg(args, torch, fga, cfg, q, k, v, keep, flops_per_step, flush, stream, dist, mode, out):
    """The metric end to end through the public API from pinned HOST buffers, on every rank at
    once (each rank its own shard; max time over ranks): per step H2D of Q/K/V and the
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
    dist.barrier()
    t_e = timed_steps(torch, e2e_step, max(3, args.steps // 2), flush, stream)
    e_ms = dist.max(sum(t_e) / len(t_e))
    h2d = 3 * q.numel() * 2 + bits.numel() * 4
    res = {"value": flops_per_step / (e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e_ms,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": q.numel() * 2, "ranks": dist.world,
           "path": "sparse_attention_host: pinned host Q/K/V + bit-packed slice mask -> H2D | "
                   "fga_compact_bits + fga_sparse_attn_fwd_ex | D2H, overlapped over 5 head slabs (the last one a "
                   "single head, its query groups in 2 runs); every rank its own shard at once, max time over ranks"}
    if dist.world > 1:
        res["h2d_bytes_per_step_per_rank"] = h2d
        res["h2d_bytes_per_step"] = h2d * (dist.world if mode != "tiles" else 1)
        res["d2h_bytes_per_step"] = q.numel() * 2 * (dist.world if mode != "tiles" else 1)
    if out is not None:
        res["max_abs_diff_vs_device_path"] = float((hout.float() - out.float().cpu()).abs().max())
    return res


def extras(args, torch, np, fga, cfg, q, k, v, keep, mask, out, kernel_ms, flush, stream, line, world,
           hbm_peak, peak_src, count):
    """Rank 0: dense denominators, K1b, builders and the oracle parity / CPU baseline on this
    rank's shard (the whole layer at N=1)."""
    from paper_2509_16518_b200 import _lib

    heads, n, d, m = cfg.heads, cfg.seq_len, cfg.head_dim, cfg.group_size
    if out is None:
        out = fga.sparse_attention(q, k, v, mask, cfg)
    # ---- K1b compaction (HBM-bound): keep bytes (or bits) read + 4*count written (+ counts)
    live = 4 * int(mask.counts.sum().item()) + 4 * mask.counts.numel()
    t_c = timed_steps(torch, lambda: fga.compact_keep(keep, m), max(3, args.steps), flush, stream)
    c_ms = sorted(t_c)[len(t_c) // 2]
    c_bytes = keep.numel() + live
    bits_dev = fga.pack_keep_bits(keep)
    t_b = timed_steps(torch, lambda: fga.compact_keep_bits(bits_dev, m, n), max(3, args.steps), flush, stream)
    b_ms = sorted(t_b)[len(t_b) // 2]
    b_bytes = bits_dev.numel() * 4 + live
    # the same kernels back to back (10 launches per event pair, each on the next of 4 rotated input
    # copies; the 181 MB of lists a launch writes exceed L2): one flushed launch reads a ~2 us event
    # clock tick against ~40 us and starts behind the flush's dirty L2 lines
    rows = keep.numel() // n
    idx_b = torch.empty((rows, n), dtype=torch.int32, device=keep.device)
    cnt_b = torch.empty(rows, dtype=torch.int32, device=keep.device)
    keeps = [keep.reshape(rows, n).clone() for _ in range(4)]
    bitss = [bits_dev.reshape(rows, -1).clone() for _ in range(4)]
    sp = stream.cuda_stream

    def batched_ms(launch, reps=5, per=10):
        for i in range(4):
            launch(i)
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in range(per):
                launch(i % 4)
            b.record(stream)
            ts.append((a, b))
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) / per for a, b in ts)[reps // 2]

    c_bat = batched_ms(lambda i: _lib.call("fga_compact", keeps[i].data_ptr(), None, rows, n, idx_b.data_ptr(), n,
                                           cnt_b.data_ptr(), 0, sp))
    b_bat = batched_ms(lambda i: _lib.call("fga_compact_bits", bitss[i].data_ptr(), rows, n, idx_b.data_ptr(), n,
                                           cnt_b.data_ptr(), 0, sp))
    del keeps, bitss, idx_b, cnt_b
    line["mask_build"] = {"kernel": "fga_compact_kernel", "ms": c_ms, "bytes": c_bytes,
                          "achieved_gbs": c_bytes / (c_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                          "frac": c_bytes / (c_ms * 1e-3) / 1e9 / hbm_peak, "peak_source": peak_src,
                          "bits_kernel": "fga_compact_bits_kernel", "bits_ms": b_ms, "bits_bytes": b_bytes,
                          "bits_achieved_gbs": b_bytes / (b_ms * 1e-3) / 1e9,
                          "bits_frac": b_bytes / (b_ms * 1e-3) / 1e9 / hbm_peak,
                          "back_to_back": {"ms": c_bat, "frac": c_bytes / (c_bat * 1e-3) / 1e9 / hbm_peak,
                                           "bits_ms": b_bat, "bits_frac": b_bytes / (b_bat * 1e-3) / 1e9 / hbm_peak,
                                           "how": "10 launches per CUDA-event pair over 4 rotated input copies, "
                                                  "no flush (each launch writes 181 MB > L2)"},
                          "layer_ms_incl_compaction": kernel_ms + min(c_ms, b_ms)}

    # ---- K1a threshold builders on the same Q/K (masks.py:94-150), each to a device mask
    from paper_2509_16518_b200 import masks as fmasks

    builders = {}
    time.sleep(0.5)  # (clocks back from any earlier power-capped leg)
    with ClockSampler(q.device.index) as clk_b:
        for name, fn in (
                ("cached_threshold_ms", lambda: fmasks.build_mask_cached_qk(q, k, cfg, 0.5 / n, device_result=True)),
                ("avg_query_topk_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
                    "avg_query_topk", top_k=count), device_result=True)),
                ("avg_query_threshold_ms", lambda: fmasks.build_mask(q, k, cfg, fmasks.MaskBuilderConfig(
                    "avg_query_threshold", tau=1.0 / d), device_result=True))):
            fn()  # (first call: workspace and list buffers from the caching allocator)
            tb = timed_steps(torch, fn, 5, flush, stream)
            builders[name] = sorted(tb)[len(tb) // 2]
    builders["clocks"] = clk_b.summary()
    builders["cached_amortised_per_iteration_ms"] = builders["cached_threshold_ms"] / 15
    line["mask_builders"] = builders

    # ---- variable-length masks (avg-query threshold builder, per-group query scales): dynamic
    #      longest-first tile scheduling vs the static stride (tail of the persistent kernel)
    line["variable_mask"] = variable_mask_leg(torch, fga, cfg, q, k, v, flush, stream)

    # ---- dense denominators on the same GPU and shard: our dense kernel + torch SDPA backends
    dense = {}
    time.sleep(0.5)  # (same starting clocks as the headline steps)
    clk_d = ClockSampler(q.device.index).__enter__()
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
        except Exception:  # backend not available for this shape
            dense[name] = None
    best = min(x for x in dense.values() if x)
    dense["best_ms"] = best
    # full mask (sparse.py:206-213): sparse_attention dispatches it to the contiguous-chunk kernel;
    # the gather kernel on the same all-keys lists for comparison (FGA_DENSE_DISPATCH=0)
    g_ = cfg.num_groups
    fidx = torch.arange(n, dtype=torch.int32, device=q.device).expand(1, heads, g_, n).contiguous()
    fmask = fga.DeviceIndexMask(1, heads, n, m, fidx, torch.full((1, heads, g_), n, dtype=torch.int32,
                                                                 device=q.device), validated=True)
    tf = timed_steps(torch, lambda: fga.sparse_attention(q, k, v, fmask, cfg), max(3, args.steps // 2), flush, stream)
    os.environ["FGA_DENSE_DISPATCH"] = "0"
    try:
        tg = timed_steps(torch, lambda: fga.sparse_attention(q, k, v, fmask, cfg), max(3, args.steps // 2), flush,
                         stream)
    finally:
        os.environ.pop("FGA_DENSE_DISPATCH", None)
    dense["full_mask_dispatched_ms"] = sorted(tf)[len(tf) // 2]
    dense["full_mask_gather_kernel_ms"] = sorted(tg)[len(tg) // 2]
    del fidx, fmask
    clk_d.__exit__(None, None, None)
    dense["clocks"] = clk_d.summary()
    dense["dense_flops"] = 4 * d * heads * n * n
    dense["shard"] = f"{heads} heads on this GPU" if world > 1 else "the whole layer"
    line["dense"] = dense
    line["speedup_vs_dense"] = best / kernel_ms

    # ---- sustained: the same launch back to back for ~1 s (no L2 flush, the board at its power
    #      cap), next to the burst number of the timed steps; last of the GPU legs, so the dense
    #      denominators, K1b and the builders above are timed at the same (burst) clocks as the
    #      headline
    n_sus = max(20, int(1000.0 / max(kernel_ms, 0.05)))
    fga.sparse_attention(q, k, v, mask, cfg)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(q.device.index) as clk_sus:
        ev0.record(stream)
        for _ in range(n_sus):
            fga.sparse_attention(q, k, v, mask, cfg)
        ev1.record(stream)
        torch.cuda.synchronize()
    sus_ms = ev0.elapsed_time(ev1) / n_sus
    line["sustained"] = {"launches": n_sus, "ms_per_launch": sus_ms,
                         "tflops": line["roofline"]["achieved"] * kernel_ms / sus_ms if "roofline" in line else None,
                         "clocks": clk_sus.summary(), "l2": "not flushed (back to back)"}
    # ---- oracle parity on >= 2 whole heads (+ bounded by --cpu-seconds); timed as the CPU
    #      baseline at N=1
    cores = host_cores()
    per_group_s = 4 * d * m * count / 25e9      # ~25 GFLOP/s per core for the NumPy port
    budget = max(cores, int(args.cpu_seconds * cores / per_group_s))
    whole = [(h, g) for h in range(min(2, heads)) for g in range(cfg.num_groups)]
    units = whole + [(h, g) for h in range(2, heads) for g in range(cfg.num_groups)][:max(0, budget - len(whole))]
    heads_used = sorted({h for h, _ in units})
    qh, kh, vh = (x[0, heads_used].float().cpu().numpy() for x in (q, k, v))
    pos = {h: i for i, h in enumerate(heads_used)}
    local_units = [(pos[h], g) for h, g in units]
    idx_rows = np.stack([mask.idx[0, h, g].cpu().numpy() for h, g in units])
    cnts = np.array([int(mask.counts[0, h, g]) for h, g in units], np.int32)
    secs, cpu_out = run_cpu_units(qh, kh, vh, idx_rows, cnts, local_units, m, cfg.scale, cores)
    rows = np.array([min(m, n - g * m) for _, g in units])
    f_sample = int(4 * d * (rows * cnts.astype(np.int64)).sum())
    err = 0.0
    gpu = out[0, heads_used].float().cpu().numpy()
    for j, (hl, g) in enumerate(local_units):
        lo, hi = g * m, min(g * m + m, n)
        err = max(err, float(np.abs(gpu[hl, lo:hi] - cpu_out[j, : hi - lo]).max()))
    line["parity"] = {"max_abs_err_vs_oracle": err, "tolerance": 2e-2, "groups_checked": len(units),
                      "whole_heads_checked": sum(1 for h in heads_used
                                                 if sum(1 for hh, _ in units if hh == h) == cfg.num_groups),
                      "output_dtype": "bf16", "oracle": "oracle.sparse_attention_group (sparse.py:138-155)"}
    if world == 1:
        cpu_val = f_sample / secs / 1e12
        full = len(units) == heads * cfg.num_groups
        line["cpu_baseline"] = {"value": cpu_val, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                                "sample": (f"{'the whole layer' if full else 'a bounded sample'}: {len(units)} query "
                                           f"groups x {count} keys over {len(heads_used)} heads, "
                                           "oracle.sparse_attention_group, one process per core"),
                                "seconds": secs, "core_seconds": secs * cores,
                                "gpu_vs_cpu_ratio": line["value"] / cpu_val}


def variable_mask_leg(torch, fga, cfg, q, k, v, flush, stream):
    """Attention on a builder-produced mask with list lengths varying ~10-50% of N per group,
    timed with the dynamic longest-first scheduler and with the static stride."""
    f = torch.tensor([0.2 + 3.8 * (g % 7) / 6 for g in range(cfg.num_groups)], device=q.device)
    qq = (q.float() * f.repeat_interleave(cfg.group_size)[: cfg.seq_len, None]).to(torch.bfloat16)
    mask = fga.build_mask(qq, k, cfg, fga.MaskBuilderConfig("avg_query_threshold", tau=1.02 / cfg.head_dim),
                          device_result=True)
    c = mask.counts.double()
    flops = fga.count_flops(cfg, mask).flops_matmul
    res = {"mask": "avg_query_threshold (tau=1.02/D) on Q scaled per group by 0.2..4.0",
           "density": float(c.mean()) / cfg.seq_len, "count_cv": float(c.std() / c.mean())}
    prev = os.environ.get("FGA_ATTN_KERNEL")
    try:
        for name, mode in (("dynamic", ""), ("static", "static")):
            os.environ["FGA_ATTN_KERNEL"] = mode
            fga.sparse_attention(q, k, v, mask, cfg)
            ts = timed_steps(torch, lambda: fga.sparse_attention(q, k, v, mask, cfg), 7, flush, stream)
            ms = sorted(ts)[len(ts) // 2]
            res[f"{name}_ms"] = ms
            res[f"{name}_tflops"] = flops / (ms * 1e-3) / 1e12
    finally:
        if prev is None:
            os.environ.pop("FGA_ATTN_KERNEL", None)
        else:
            os.environ["FGA_ATTN_KERNEL"] = prev
    # ideal: the pairs spread evenly over the SMs at the dynamic run's pair rate -> the tail is
    # the time the last CTAs run alone; static / dynamic shows what the scheduler recovers
    res["static_over_dynamic"] = res["static_ms"] / res["dynamic_ms"]
    # per-CTA timeline of one launch each (fga_sparse_attn_fwd_timed, %globaltimer at CTA start / end):
    # tail fraction = longest CTA / mean CTA (1.0 = perfectly balanced)
    from paper_2509_16518_b200 import _lib

    sms = torch.cuda.get_device_properties(q.device).multi_processor_count
    buf = torch.zeros(2 * sms, dtype=torch.int64, device=q.device)
    o = torch.empty_like(q)
    shp = _lib.shape(*cfg.dims, cfg.group_size, cfg.scale)
    for name, flags, order in (("dynamic", 0, mask.tile_order(cfg)), ("static", _lib.FGA_ATTN_STATIC, None)):
        for _ in range(2):  # the second launch is the one kept (warm)
            flush.zero_()
            buf.zero_()
            _lib.call("fga_sparse_attn_fwd_timed", q.data_ptr(), k.data_ptr(), v.data_ptr(), mask.idx.data_ptr(),
                      mask.stride, mask.counts.data_ptr(), o.data_ptr(), _lib.FGA_OUT_BF16, None, shp, 0, -1,
                      None if order is None else order.data_ptr(), None, flags, buf.data_ptr(), buf.numel(),
                      stream.cuda_stream)
        torch.cuda.synchronize()
        t = buf.view(-1, 2).double()
        t = t[t[:, 1] > 0]
        busy = (t[:, 1] - t[:, 0]) / 1e6
        res[f"{name}_cta_tail_fraction"] = float(busy.max() / busy.mean())
        res[f"{name}_cta_ms"] = {"mean": float(busy.mean()), "max": float(busy.max()), "min": float(busy.min()),
                                 "makespan": float((t[:, 1].max() - t[:, 0].min()) / 1e6), "ctas": int(t.shape[0])}
    return res


def c5_sweep(args, torch, fga, _lib, shard, dist, dev, flush, stream, world, rank):
    """BASELINE configs[4]: Wan 14B at 720p head-sharded over the GPUs, density 10-90%:
    layer latency (max over ranks), TFLOP/s and speed-up over cuDNN dense on the same shard."""
    heads, n, d, m, desc = CONFIGS["c5"]
    cfg = fga.AttnConfig(1, heads, n, d, group_size=m, precision="bf16")
    h0, h1 = shard.head_blocks(heads, world)[rank]
    lcfg = fga.AttnConfig(1, h1 - h0, n, d, group_size=m, precision="bf16")
    gen = torch.Generator(device=dev).manual_seed(4321 + args.seed)
    full = [torch.randn(cfg.dims, device=dev, generator=gen).to(torch.bfloat16) for _ in range(3)]
    lq, lk, lv = (x[:, h0:h1].contiguous() for x in full)
    del full
    from torch.nn.attention import SDPBackend, sdpa_kernel

    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        torch.nn.functional.scaled_dot_product_attention(lq, lk, lv)
        td = timed_steps(torch, lambda: torch.nn.functional.scaled_dot_product_attention(lq, lk, lv), 5, flush, stream)
    dense_ms = dist.max(sorted(td)[len(td) // 2])
    rows = []
    for dens in SWEEP:
        keep = make_keep(torch, _lib, cfg, dens, args.seed, dev)[:, h0:h1].contiguous()
        mask = fga.compact_keep(keep, m)
        mask.validated = True
        del keep
        fga.sparse_attention(lq, lk, lv, mask, lcfg)
        torch.cuda.synchronize()
        dist.barrier()
        ts = timed_steps(torch, lambda: fga.sparse_attention(lq, lk, lv, mask, lcfg), 5, flush, stream)
        ms = dist.max(sorted(ts)[len(ts) // 2])
        count = max(1, round(dens * n))
        flops = 4 * d * heads * n * count
        rows.append({"density": dens, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12, "speedup_vs_cudnn": dense_ms / ms})
        del mask
    return {"workload": desc, "n_gpus": world, "heads_per_gpu": h1 - h0, "cudnn_dense_ms": dense_ms, "rows": rows}


def main():
    args = parse()
    if args.cpu_worker:
        _cpu_pool_main(args.cpu_worker)
        return
    if args.ref_worker:
        _ref_worker_main(args.ref_worker)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        reference_arm(args)
        return
    if args.dry_run:
        dry_run(args)
        return
    ours(args)


if __name__ == "__main__":
    main()
