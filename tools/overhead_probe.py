"""Host overhead of a call vs the device time of its captured step (logreg).
Diagnostic only.

    python tools/overhead_probe.py
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402
from paper_1605_02688_b200 import native  # noqa: E402


def main():
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    g = C.build_logreg(T)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    x, y = C.inputs_logreg()
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(5):
        f.call_device(xd, yd)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        f.call_device(xd, yd)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"call_device: host {1e6 * (t1 - t0) / n:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / n:.1f} us/call")
    plan = next(iter(f._plans.values()))
    st = f._stream
    e0, e1 = lib.event_create(), lib.event_create()
    lib.event_record(e0, st)
    for _ in range(n):
        lib.graph_launch(plan.graph, st)
    lib.event_record(e1, st)
    lib.stream_sync(st)
    print(f"graph replay back-to-back: {1e3 * lib.elapsed_ms(e0, e1) / n:.2f} us/step (device)")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        f.call_device(xd, yd)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def host_calls():
    """f(x, y) with NumPy arrays (the public call): where its time goes."""
    torch.cuda.set_device(0)
    g = C.build_logreg(T)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    x, y = C.inputs_logreg()
    for _ in range(5):
        f(x, y)
    n = 300
    t0 = time.perf_counter()
    for _ in range(n):
        f(x, y)
    t1 = time.perf_counter()
    print(f"f(x, y) host arrays: {1e6 * (t1 - t0) / n:.1f} us/call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        f(x, y)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "host":
    host_calls()
