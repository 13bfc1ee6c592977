"""bench.py's multi-GPU host logic on the CPU (gloo, no kernels): ``--gpus N`` self-launches N
ranks under torch.distributed.run, the head-sharded (c4) and tile-sharded (c2 on 8) partitions,
the max-over-ranks reduction and the validation all-gather."""

import json
import os
import subprocess
import sys


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None, timeout=240):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=dict(os.environ, **(env or {})), cwd=ROOT)
    return r


def last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_self_launch_two_ranks_head_sharded():
    r = run_bench("--gpus", "2", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    line = last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["shard"] == "heads" and line["config"]["config"] == "c4"
    assert line["head_blocks"] == [[0, 20], [20, 40]]
    assert line["gather_ok"] is True and line["max_rank_allreduce"] == 1.0


def test_uneven_heads_fall_back_to_tile_ranges():
    r = run_bench("--gpus", "8", "--dry-run", "--config", "c2")
    assert r.returncode == 0, r.stderr[-2000:]
    line = last_json(r.stdout)
    assert line["n_gpus"] == 8 and line["shard"] == "tiles"
    rng = line["tile_ranges"]
    assert rng[0][0] == 0 and rng[-1][1] == 12 * 256 and all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
    assert line["gather_ok"] is True


def test_world_size_must_match_gpus():
    r = run_bench("--gpus", "4", "--dry-run", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in (r.stderr + r.stdout)
