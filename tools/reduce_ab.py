"""CAReduce timing over a 16384^2 fp32 matrix (CUDA events, median of reps;
never a bench number).  python tools/reduce_ab.py [op ...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1605_02688_b200 as T
    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    X = torch.randn(16384, 16384, device="cuda")
    v = T.matrix("X", dtype="float32")
    ops = sys.argv[1:] or ["sum", "max", "argmax"]
    for name in ops:
        build = getattr(T, name)
        for ax in ((0,), (1,), None):
            f = T.compile([v], build(v, axis=ax))
            for _ in range(3):
                f.call_device(X)
            ts = []
            for _ in range(15):
                e0, e1 = lib.event_create(), lib.event_create()
                lib.event_record(e0, f._stream)
                f.call_device(X)
                lib.event_record(e1, f._stream)
                lib.stream_sync(f._stream)
                ts.append(lib.elapsed_ms(e0, e1))
            ms = statistics.median(ts)
            print(f"{name} axis={ax}: {ms * 1e3:.1f} us  {X.numel() * 4 / ms / 1e6:.0f} GB/s  (min {min(ts) * 1e3:.1f})")


if __name__ == "__main__":
    main()
