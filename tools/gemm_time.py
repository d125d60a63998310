"""Time one device GEMM shape in one mode (CUDA events, mean of 10 after 3 warm-ups)."""
import sys
import torch
import paper_1605_02688_b200 as T
M, N, K = (int(v) for v in sys.argv[1:4])
mode = sys.argv[4] if len(sys.argv) > 4 else "auto"
a = torch.randn(M, K, device="cuda")
b = torch.randn(K, N, device="cuda")
va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
f = T.compile([va, vb], T.dot(va, vb), gemm_mode=mode)
for _ in range(3):
    f.call_device(a, b)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    f.call_device(a, b)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"{M}x{N}x{K} {mode}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TF/s", flush=True)
