"""Interleaved timing of the skinny-N GEMM variants on the MLP's h2.W3 shape
(diagnostic)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from paper_1605_02688_b200 import native  # noqa: E402

torch.cuda.set_device(0)
lib = native.device_library(0)
a = torch.randn(8192, 4096, device="cuda")
b = torch.randn(4096, 10, device="cuda")
va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
f = T.compile([va, vb], T.dot(va, vb), cuda_graph=False)
res = {}
for rep in range(5):
    for var in ("0", "3"):
        os.environ["TX_RD_VARIANT"] = var
        for _ in range(2):
            f.call_device(a, b)
        e0, e1 = lib.event_create(), lib.event_create()
        lib.event_record(e0, f._stream)
        for _ in range(20):
            f.call_device(a, b)
        lib.event_record(e1, f._stream)
        lib.stream_sync(f._stream)
        res.setdefault(var, []).append(lib.elapsed_ms(e0, e1) / 20)
for var, v in res.items():
    ms = statistics.median(v)
    print(f"variant {var}: {ms * 1e3:.1f} us  {8192 * 4096 * 4 / (ms * 1e-3) / 1e9:.0f} GB/s")
