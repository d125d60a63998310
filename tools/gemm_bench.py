"""TF32 GEMM microbenchmark over the MLP shapes and layouts (CUDA events on
the VM stream; correctness vs an fp64 product on a sample of rows).

    TX_GEMM_CG=1|2 python tools/gemm_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from paper_1605_02688_b200 import native  # noqa: E402

SHAPES = [  # (name, M, N, K, a_transposed, b_transposed)
    ("G1 x.W1", 8192, 4096, 784, False, False),
    ("G2 h1.W2", 8192, 4096, 4096, False, False),
    ("G6 dz2.W2T", 8192, 4096, 4096, False, True),
    ("G7 h1T.dz2", 4096, 4096, 8192, True, False),
    ("G8 xT.dz1", 784, 4096, 8192, True, False),
    ("TT", 4096, 4096, 4096, True, True),
    ("8192^3 NN", 8192, 8192, 8192, False, False),
    # diagnostics for the short-K forward GEMM
    ("G1kmaj x.W1(K-major)", 8192, 4096, 784, False, True),
    ("K1568 NN", 8192, 4096, 1568, False, False),
    ("K3136 NN", 8192, 4096, 3136, False, False),
    ("K800kk", 8192, 4096, 800, False, True),
    # LSTM PTB medium per-step products (batch 20, hidden 600, vocabulary 10000)
    ("L1 x.Wx", 20, 2400, 600, False, False),
    ("L2 h.Wo", 20, 10000, 600, False, False),
    ("L3 dy.WoT", 20, 600, 10000, False, True),
    ("L4 hT.dy", 600, 10000, 20, True, False),
    ("L5 dz.WxT", 20, 600, 2400, False, True),
    ("L6 xT.dz", 600, 2400, 20, True, False),
]


def bench_fn(lib, f, args, reps=10):
    f.call_device(*args, sync=True)
    for _ in range(3):
        f.call_device(*args)
    ev = [(lib.event_create(), lib.event_create()) for _ in range(reps)]
    for e0, e1 in ev:
        lib.event_record(e0, f._stream)
        f.call_device(*args)
        lib.event_record(e1, f._stream)
    lib.stream_sync(f._stream)
    return sorted(lib.elapsed_ms(e0, e1) for e0, e1 in ev)[reps // 2]


def epilogues(lib):
    """The MLP's fused forward (tanh(b + x.W)) and backward (dH * g) GEMMs."""
    M, N = 8192, 4096
    for K in (784, 4096):
        x = torch.randn(M, K, device="cuda")
        w = torch.randn(K, N, device="cuda") / K ** 0.5
        bias = torch.randn(N, device="cuda")
        vx, vw, vb = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32"), T.vector("b", dtype="float32")
        h = T.tanh(T.dot(vx, vw) + vb)
        for fuse in (True, False):
            f = T.compile([vx, vw, vb], [h], exclude=() if fuse else ("fuse_gemm_epilogue",))
            ms = bench_fn(lib, f, (x, w, bias))
            print(f"fwd K={K} fused={fuse}: {ms:.3f} ms ({2 * M * N * K / ms / 1e9:.1f} TFLOP/s incl. epilogue)", flush=True)
    dz = torch.randn(M, N, device="cuda")
    w2 = torch.randn(N, N, device="cuda")
    g = torch.randn(M, N, device="cuda")
    vd, vw2, vg = T.matrix("dz", dtype="float32"), T.matrix("w2", dtype="float32"), T.matrix("g", dtype="float32")
    for fuse in (True, False):
        f = T.compile([vd, vw2, vg], T.dot(vd, T.transpose(vw2)) * vg, exclude=() if fuse else ("fuse_gemm_epilogue",))
        ms = bench_fn(lib, f, (dz, w2, g))
        print(f"bwd dH*g fused={fuse}: {ms:.3f} ms ({2 * M * N * N / ms / 1e9:.1f} TFLOP/s incl. epilogue)", flush=True)


def cublas_ms(A, B, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(3):
        A @ B
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        A @ B
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    torch.backends.cuda.matmul.allow_tf32 = False
    return sorted(ts)[reps // 2]


def main():
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    cg = os.environ.get("TX_GEMM_CG", "2")
    only = sys.argv[1:]
    for name, M, N, K, ta, tb in SHAPES:
        if only and name.split()[0] not in only:
            continue
        a = torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")
        b = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
        va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
        f = T.compile([va, vb], T.dot(T.transpose(va) if ta else va, T.transpose(vb) if tb else vb))
        out = f.call_device(a, b, sync=True)
        for _ in range(3):
            f.call_device(a, b)
        ev = [(lib.event_create(), lib.event_create()) for _ in range(10)]
        for e0, e1 in ev:
            lib.event_record(e0, f._stream)
            f.call_device(a, b)
            lib.event_record(e1, f._stream)
        lib.stream_sync(f._stream)
        ms = sorted(lib.elapsed_ms(e0, e1) for e0, e1 in ev)[len(ev) // 2]
        out = f.call_device(a, b, sync=True)
        A = (a.T if ta else a)
        B = (b.T if tb else b)
        rows = torch.randint(0, M, (64,), device="cuda")
        ref = (A[rows].double() @ B.double())
        bound = (A[rows].abs().double() @ B.abs().double())
        err = ((out[rows].double() - ref).abs() / (bound + 1e-30)).max().item()
        tf = 2 * M * N * K / (ms * 1e-3) / 1e12
        cb = cublas_ms(A, B) if not only else float("nan")
        print(f"CG={cg} {name:12s} M={M} N={N} K={K}: {ms:.3f} ms {tf:7.1f} TFLOP/s  max err/bound {err:.2e}"
              f"   | cuBLAS TF32 same layout {cb:.3f} ms {2 * M * N * K / (cb * 1e-3) / 1e12:7.1f} TFLOP/s", flush=True)
    if not only:
        epilogues(lib)


if __name__ == "__main__":
    main()
