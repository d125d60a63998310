"""MLP B=8192 step time per GEMM mode (diagnostic; bench.py reports the same in extra)."""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1605_02688_b200 as T
from oracle import configs as C
from paper_1605_02688_b200 import native
lib = native.device_library(0)
for mode in (sys.argv[1:] or ["auto", "3xtf32"]):
    f, ms, cost = bench.bench_mlp(T, C, 8192, 10, 3, lambda: lib, gemm_mode=mode)
    print(mode, f"{statistics.median(ms):.3f} ms/step", [round(v, 3) for v in ms], flush=True)
