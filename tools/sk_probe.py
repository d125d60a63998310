"""Stream-K GEMM probe (diagnostic): correctness of a few shapes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402

torch.cuda.set_device(0)
for (M, N, K) in [(256, 512, 256), (4096, 4096, 1024), (784, 4096, 2048)]:
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(K, N, device="cuda")
    va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    f = T.compile([va, vb], T.dot(va, vb))
    out = f.call_device(a, b, sync=True)
    ref = (a.double() @ b.double())
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    print(M, N, K, "max rel err", err, flush=True)
