"""bench.py launch plumbing on CPU: `--gpus N` outside a launcher self-spawns N ranks
(torch.distributed.run, gloo in --dry-run), and both arms print the same metric string."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_self_spawn_two_ranks():
    d = _run("--gpus", "2", "--dry-run")
    assert d["n_gpus"] == 2 and d["ranks"] == [0, 1]


def test_single_rank_default():
    d = _run("--dry-run")
    assert d["n_gpus"] == 1 and d["ranks"] == [0]


def test_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_same_metric_both_arms():
    a = _run("--dry-run")
    b = _run("--dry-run", "--impl", "reference")
    assert a["metric"] == b["metric"]
    sys.path.insert(0, ROOT)
    import bench
    assert bench.METRIC == a["metric"]
