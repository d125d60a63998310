"""A/B of the 1-rank data-parallel MLP step at the config-5 batch (diagnostic)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import bench
import paper_1605_02688_b200 as T
from oracle import configs as C
from paper_1605_02688_b200 import native
from paper_1605_02688_b200.dp import DataParallel
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
lib = native.device_library(0)
for _ in range(2):
    for dpm in (True, False):
        dp = DataParallel(world_size=1, rank=0) if dpm else None
        f, ms, cost = bench.bench_mlp(T, C, 65536, 5, 3, lambda: lib, dp=dp, n_global=65536)
        import statistics
        print("dp" if dpm else "plain", f"{statistics.median(ms):.3f} ms/step", [round(v, 2) for v in ms], flush=True)
dist.destroy_process_group()
