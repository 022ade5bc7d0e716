"""bench.py's multi-GPU launch contract (CPU only, gloo dry run): `python
bench.py --gpus N` outside torchrun starts N ranks itself and every rank takes
the distributed arm; `--gpus 1` stays a single process."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ, RLRA_B200_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], env=env, capture_output=True,
                         text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]


def test_gpus_2_starts_two_ranks_on_the_dist_arm():
    lines = _run("--gpus", "2")
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["arm"] == "dist" and x["world"] == 2 for x in lines)


def test_gpus_1_is_one_process():
    lines = _run("--gpus", "1")
    assert lines == [{"dryrun": True, "arm": "single", "rank": 0, "world": 1}]


def test_torchrun_command_matches_the_driver_launch():
    sys.path.insert(0, REPO)
    import bench

    cmd = bench.torchrun_cmd(["--gpus", "8", "--steps", "3"], 8, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "8", "--steps", "3"][-3:]
