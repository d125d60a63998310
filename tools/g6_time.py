"""Time the MLP's big products by layout (G2 h1.W2, G6 dz2.W2^T, G7 h1^T.dz2) under env knobs (diagnostic)."""
import torch
import paper_1605_02688_b200 as T
M = N = K = 4096
B = 8192
a = torch.randn(B, K, device="cuda")
w = torch.randn(K, N, device="cuda")
va, vw = T.matrix("a", dtype="float32"), T.matrix("w", dtype="float32")
cases = (("G2 a.w", T.dot(va, vw), (a, w)), ("G6 a.w^T", T.dot(va, T.transpose(vw)), (a, w)),
         ("G7 a^T.b", T.dot(T.transpose(va), vw), (a, torch.randn(B, N, device="cuda"))))
for name, expr, args in cases:
    f = T.compile([va, vw], expr)
    for _ in range(3):
        f.call_device(*args)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f.call_device(*args)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name}: {ms * 1e3:.1f} us  {2 * 8192 * 4096 * 4096 / ms / 1e9:.1f} TF/s", flush=True)
