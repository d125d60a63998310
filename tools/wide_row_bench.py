"""Softmax + cross-entropy forward and gradient over wide rows, row fusion on
vs off (CUDA events, never a bench number).  TX_ROW_WIDE_T picks the threads
per row of the block-per-row form."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1605_02688_b200 as T
    from bench import time_device_block
    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    for N, K in ((20, 10000), (800, 10000), (256, 4096), (4096, 1000)):
        z = T.matrix("z", dtype="float32")
        y = T.matrix("y", dtype="float32")
        m = T.max(z, axis=1)
        e = T.exp(z - T.dimshuffle(m, (0, "x")))
        p = e / T.dimshuffle(T.sum(e, axis=1), (0, "x"))
        cost = -T.sum(y * T.log(p)) / float(N)
        (gz,) = T.grad(cost, [z])
        for rf in (False, True):
            f = T.compile([z, y], [cost, gz], row_fusion=rf)
            zv = torch.randn(N, K, device="cuda")
            yv = torch.zeros(N, K, device="cuda")
            yv[:, 3] = 1
            for _ in range(3):
                f.call_device(zv, yv)
            us = time_device_block(lambda: f.call_device(zv, yv), lib, f._stream, 50) * 1e3
            print(f"N={N} K={K} row_fusion={rf} T={os.environ.get('TX_ROW_WIDE_T', '1024')}: {us:.1f} us "
                  f"({3 * N * K * 4 / us / 1e3:.0f} GB/s of z, y read + gz written)")


if __name__ == "__main__":
    main()
