"""Time dot+add_aux_bias vs unfused at small shapes (diagnostic)."""
import sys
import numpy as np
import torch
import paper_1605_02688_b200 as T
for (M, N, K) in [(20, 800, 200), (20, 2400, 600), (300, 520, 784)]:
    vx, vw = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32")
    vg, vb = T.matrix("g", dtype="float32"), T.vector("b", dtype="float32")
    expr = (vg + T.dot(vx, vw)) + vb
    x = torch.randn(M, K, device="cuda"); w = torch.randn(K, N, device="cuda")
    g = torch.randn(M, N, device="cuda"); b = torch.randn(N, device="cuda")
    for ex in ((), ("fuse_gemm_epilogue",)):
        f = T.compile([vx, vw, vg, vb], expr, exclude=ex)
        for _ in range(3):
            f.call_device(x, w, g, b)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            f.call_device(x, w, g, b)
        e.record(); torch.cuda.synchronize()
        print(M, N, K, "fused" if not ex else "unfused", round(s.elapsed_time(e) / 50 * 1e3, 1), "us", flush=True)
