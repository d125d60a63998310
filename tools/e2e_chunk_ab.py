"""Config-2 end-to-end (pinned host tensors) under TX_CHUNK_MB (diagnostic)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1605_02688_b200 as T
from oracle import configs as C
g = C.build_ew(T)
f = T.compile(g["inputs"], g["outputs"])
dt, bi, bo, dtn = bench.bench_ew_e2e(f, steps=5)
print(f"chunk {os.environ.get('TX_CHUNK_MB', '32')} MB: pinned {dt * 1e3:.1f} ms/step = {(bi + bo) / dt / 1e9:.1f} GB/s; "
      f"numpy {dtn * 1e3:.1f} ms = {(bi + bo) / dtn / 1e9:.1f} GB/s", flush=True)
