"""Interleaved A/B timing of one GEMM shape under two environment settings
(the tcgen05 path reads its TX_GEMM_* switches at every launch), so box-level
clock drift hits both arms equally.  Diagnostic only.

    python tools/gemm_ab.py G8 TX_GEMM_NO3D=1
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from paper_1605_02688_b200 import native  # noqa: E402
from tools.gemm_bench import SHAPES  # noqa: E402


def main():
    name, env = sys.argv[1], sys.argv[2:]
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    _, M, N, K, ta, tb = next(s for s in SHAPES if s[0].split()[0] == name)
    a = torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
    va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    f = T.compile([va, vb], T.dot(T.transpose(va) if ta else va, T.transpose(vb) if tb else vb), cuda_graph=False)
    kv = [e.split("=", 1) for e in env]

    def run(on, reps=20):
        for k, v in kv:
            if on:
                os.environ[k] = v
            else:
                os.environ.pop(k, None)
        for _ in range(3):
            f.call_device(a, b)
        e0, e1 = lib.event_create(), lib.event_create()
        lib.event_record(e0, f._stream)
        for _ in range(reps):
            f.call_device(a, b)
        lib.event_record(e1, f._stream)
        lib.stream_sync(f._stream)
        return lib.elapsed_ms(e0, e1) / reps

    A, B = [], []
    for _ in range(6):
        A.append(run(False))
        B.append(run(True))
    fl = 2 * M * N * K
    ma, mb = statistics.median(A), statistics.median(B)
    print(f"{name} M={M} N={N} K={K}: default {ma * 1e3:.1f} us ({fl / ma / 1e9:.0f} TFLOP/s) | "
          f"{' '.join(env)} {mb * 1e3:.1f} us ({fl / mb / 1e9:.0f} TFLOP/s)")


if __name__ == "__main__":
    main()
