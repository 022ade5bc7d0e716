"""Run the multi-GPU bench entry (distributed.bench_main) on a 1-rank NCCL group:
the code path torchrun --nproc-per-node N takes for N > 1 (minus the peers)."""
import os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
from paper_2002_07138_b200 import distributed as D
D.INTERIOR = os.environ.get("INTERIOR", "tslu_always")
args = types.SimpleNamespace(config=os.environ.get("CONFIG", "C2"), v=None, steps=3, warmup=1)
sys.exit(D.bench_main(args))
