"""Where does the host-array call's time go?  (diagnostic, not a bench number)

    python tools/e2e_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402
from paper_1605_02688_b200 import native  # noqa: E402


def tm(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    nb = 1 << 30
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = lib.stream_create()
    print("torch copy_ H2D GB/s", nb / tm(lambda: d.copy_(h, non_blocking=True)) / 1e9)

    def libcopy():
        lib.memcpy(d.data_ptr(), h.data_ptr(), nb, 0, s)
        lib.stream_sync(s)
    print("lib memcpy H2D GB/s (torch-pinned src)", nb / tm(libcopy) / 1e9)

    def libcopy_chunks():
        for o in range(0, nb, 32 << 20):
            lib.memcpy(d.data_ptr() + o, h.data_ptr() + o, 32 << 20, 0, s)
        lib.stream_sync(s)
    print("lib memcpy H2D 32MB chunks GB/s", nb / tm(libcopy_chunks) / 1e9)
    t0 = time.perf_counter()
    x = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    print("pinned alloc 1GiB s", time.perf_counter() - t0)
    del x
    t0 = time.perf_counter()
    x = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    print("pinned alloc 1GiB (cached) s", time.perf_counter() - t0)
    del x, h, d

    g = C.build_ew(T)
    f = T.compile(g["inputs"], g["outputs"])
    n = 1 << 28
    host = [torch.randn(n, dtype=torch.float32).pin_memory() for _ in range(4)]
    for _ in range(2):
        f(*host)
    for _ in range(3):
        t0 = time.perf_counter()
        out = f(*host)
        print("f(*host) s", time.perf_counter() - t0)
    f.pipelined = False
    f(*host)
    for _ in range(2):
        t0 = time.perf_counter()
        out = f(*host)
        print("f(*host) unpipelined s", time.perf_counter() - t0)
    del out
    # pipeline stage timing with events
    f.pipelined = True
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    f(*host)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(15)


if __name__ == "__main__":
    main()
