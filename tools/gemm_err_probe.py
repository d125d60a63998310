"""Error statistics of the device GEMM modes vs float64 and vs NumPy sgemm.
Env knobs (TX_3X_ORDER, TX_GEMM_FORCE_SPLITS) are read by the library."""
import sys
import numpy as np
import paper_1605_02688_b200 as T

rng = np.random.default_rng(0)
modes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["3xtf32"]
shapes = [(1024, 4096, 128), (1024, 1024, 1024), (2048, 2048, 4096), (784, 1024, 8192)]
for (M, N, K) in shapes:
    for dist in ("normal", "uniform"):
        if dist == "normal":
            a = rng.standard_normal((M, K)).astype(np.float32)
            b = rng.standard_normal((K, N)).astype(np.float32)
        else:
            a = rng.random((M, K), dtype=np.float32)
            b = rng.random((K, N), dtype=np.float32)
        A, B = a.astype(np.float64), b.astype(np.float64)
        want = A @ B
        bound = np.abs(A) @ np.abs(B)
        row = {"shape": (M, N, K), "dist": dist}
        sg = (a @ b).astype(np.float64)
        e = sg - want
        row["sgemm"] = ["%.2e" % float((np.abs(e) / bound).max()), "%.2e" % (float(np.mean(e * np.sign(want))) / float(np.mean(np.abs(want))))]
        for mode in modes:
            va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
            f = T.compile([va, vb], T.dot(va, vb), gemm_mode=mode)
            got = f(a, b).astype(np.float64)
            e = got - want
            row[mode] = ["%.2e" % float((np.abs(e) / bound).max()),
                         "%.2e" % (float(np.mean(e * np.sign(want))) / float(np.mean(np.abs(want)))),
                         "%.2e" % (float(np.sqrt(np.mean(e ** 2))) / float(np.sqrt(np.mean(want ** 2))))]
        print(row, flush=True)

if "--time" in sys.argv:
    import torch
    for (M, N, K) in [(8192, 4096, 4096), (8192, 4096, 784), (4096, 4096, 8192), (784, 4096, 8192)]:
        a = torch.randn(M, K, device="cuda")
        b = torch.randn(K, N, device="cuda")
        row = {"shape": (M, N, K)}
        for mode in modes:
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
            row[mode] = {"ms": round(ms, 3), "tflops": round(2 * M * N * K / ms / 1e9, 1)}
        print(row, flush=True)
