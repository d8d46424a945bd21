"""bench.py's multi-GPU launch path on CPU: `bench.py --gpus 2 --dry-run` must spawn two ranks by
itself (torch.distributed.run on 127.0.0.1, gloo), give each rank its batch shard of the headline
conv2d, and report the max-over-ranks timed region on rank 0 (one process per GPU,
no collective on the compute path)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "5",
                        "--warmup", "3", *extra], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints
    return json.loads(lines[0])


def test_gpus2_spawns_two_ranks_weak_shards():
    line = _run()
    assert line["dry_run"] and line["n_gpus"] == 2 and line["config"]["backend"] == "gloo"
    ranks = sorted(line["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == [0, 1]
    # weak: a BASELINE-sized shard (16 images of the 58x58x64 layer) per rank, global batch 32
    assert [r["op"]["I"] for r in ranks] == [[16, 64, 58, 58], [16, 64, 58, 58]]
    assert line["scaling"] == "weak" and line["config"]["batch"]["global"] == 32
    assert line["config"]["batch"]["rank_ranges"] == [[0, 16], [16, 32]]
    # the timed region is the max over ranks (rank 1's placeholder step is the longer one)
    assert line["ms_per_step"] * line["steps"] == pytest.approx(max(r["ms"] for r in ranks))
    assert ranks[1]["ms"] > ranks[0]["ms"]


def test_gpus2_strong_splits_the_batch():
    line = _run("--strong")
    ranks = sorted(line["ranks"], key=lambda r: r["rank"])
    assert [r["op"]["I"][0] for r in ranks] == [8, 8]  # 16 images split 2 ways
    assert line["scaling"] == "strong" and line["config"]["batch"]["global"] == 16
    assert sum(r["flops"] for r in ranks) == pytest.approx(2 * 16 * 64 * 56 * 56 * 64 * 9)
