"""bench.py's multi-GPU arm (dist_arm: row shards, NCCL) on a 1-rank group --
the code path torchrun --nproc-per-node N takes for N > 1, minus the peers.
usage: [CONFIG=C2|C5] [INTERIOR=tslu|gather|tslu_always] python tools/dist_bench_smoke.py"""
import os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
env = dict(os.environ, RLRA_B200_BENCH_DIST="1", RANK="0", WORLD_SIZE="1", LOCAL_RANK="0",
           MASTER_ADDR="127.0.0.1", MASTER_PORT="29533",
           RLRA_B200_DIST_INTERIOR=os.environ.get("INTERIOR", "tslu"))
cmd = [sys.executable, os.path.join(root, "bench.py"), "--steps", "5", "--warmup", "3",
       "--config", os.environ.get("CONFIG", "C2")]
sys.exit(subprocess.call(cmd, env=env))
