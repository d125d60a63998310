"""Time the MLP forward layer product h = tanh(b + x.W) (G1: 8192 x 4096 x 784,
bias+tanh epilogue) and its plain form under env knobs (diagnostic).

    [TX_GEMM_DBG_NOSTORE=1] python tools/g1_time.py [M N K]
"""
import sys
import torch
import paper_1605_02688_b200 as T
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 4096, 784)
x = torch.randn(M, K, device="cuda")
w = torch.randn(K, N, device="cuda") / K ** 0.5
b = torch.randn(N, device="cuda")
vx, vw, vb = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32"), T.vector("b", dtype="float32")
for name, expr, args in (("dot", T.dot(vx, vw), (x, w)), ("dot+bias+tanh", T.tanh(T.dot(vx, vw) + vb), (x, w, b))):
    ins = [vx, vw] + ([vb] if len(args) == 3 else [])
    f = T.compile(ins, expr)
    for _ in range(3):
        f.call_device(*args)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f.call_device(*args)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"{M}x{N}x{K} {name}: {ms * 1e3:.1f} us  {2 * M * N * K / ms / 1e9:.1f} TF/s", flush=True)
