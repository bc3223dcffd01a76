"""bench.py's launch path on a CPU box: `--gpus N` without torchrun starts N ranks itself (torch.distributed.run on
127.0.0.1), the ranks rendezvous (gloo here, NCCL on a GPU box) and rank 0 alone prints one JSON line with n_gpus = N."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    if env:
        e.update(env)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True, timeout=300, env=e)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout          # exactly one JSON line, from rank 0
    return json.loads(lines[0])


def test_gpus_2_self_launches_two_ranks():
    d = _run(["--gpus", "2", "--dry-launch", "--frames-per-rank", "3"])
    assert d["dry_launch"] and d["n_gpus"] == 2 and d["ranks_seen"] == 2
    assert d["max_over_ranks"] == 2.0           # the timing rule's reduction: MAX over ranks
    assert d["frames_assigned"] == 6            # 3 frames per rank, a partition over the ranks


def test_single_rank_dry_launch_needs_no_spawn():
    d = _run(["--dry-launch"])
    assert d["n_gpus"] == 1 and d["ranks_seen"] == 1
