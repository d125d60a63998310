"""3xTF32 time of the MLP's G2 product under env knobs (diagnostic)."""
import torch
import paper_1605_02688_b200 as T
a = torch.randn(8192, 4096, device="cuda")
w = torch.randn(4096, 4096, device="cuda")
va, vw = T.matrix("a", dtype="float32"), T.matrix("w", dtype="float32")
f = T.compile([va, vw], T.dot(va, vw), gemm_mode="3xtf32")
for _ in range(2):
    f.call_device(a, w)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    f.call_device(a, w)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"3xtf32 8192x4096x4096: {ms * 1e3:.1f} us  {2 * 8192 * 4096 * 4096 / ms / 1e9:.1f} TF/s fp32-equivalent", flush=True)
