"""Time G8-style products (A transposed view) under env knobs (diagnostic)."""
import sys
import torch
import paper_1605_02688_b200 as T
M, N, K = (int(v) for v in sys.argv[1:4])
a = torch.randn(K, M, device="cuda")   # A = a^T (MN-major)
b = torch.randn(K, N, device="cuda")
va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
f = T.compile([va, vb], T.dot(T.transpose(va), vb))
for _ in range(3):
    f.call_device(a, b)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    f.call_device(a, b)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 20
print(f"{M}x{N}x{K} (A^T): {ms * 1e3:.1f} us  {2 * M * N * K / ms / 1e9:.1f} TF/s", flush=True)
