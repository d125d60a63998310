"""Cost of the fused epilogue kinds on the G1 product (8192 x 4096 x 784) via
the C ABI: plain, +bias, +bias+tanh, TMA-store off (diagnostic)."""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1605_02688_b200 import native
lib = native.device_library(0)
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 4096, 784)
a = torch.randn(M, K, device="cuda")
b = torch.randn(K, N, device="cuda") / K ** 0.5
bias = torch.randn(N, device="cuda")
c = torch.empty(M, N, device="cuda")
mk = native.make_tensor
ta, tb, tc = mk(a.data_ptr(), "float32", (M, K), (K, 1)), mk(b.data_ptr(), "float32", (K, N), (N, 1)), mk(c.data_ptr(), "float32", (M, N), (N, 1))
wsb = lib.gemm_workspace(ta, tb, tc)
ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for name, kind in (("none", native.EPI_NONE), ("bias", native.EPI_BIAS), ("bias_tanh", native.EPI_BIAS_TANH)):
    e = native.TxEpilogue()
    e.kind = kind
    if kind != native.EPI_NONE:
        e.aux = mk(bias.data_ptr(), "float32", (N,), (1,))
    run = lambda: lib.check(lib.lib.tx_gemm(ta, tb, tc, ctypes.byref(e), native.GEMM_AUTO, ctypes.c_void_p(ws.data_ptr()), wsb, ctypes.c_void_p(st)))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(20):
        run()
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 20
    print(f"{M}x{N}x{K} {name}: {ms * 1e3:.1f} us", flush=True)
