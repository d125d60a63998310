"""Device ms/step of one workload (for A/B runs under env toggles; never a
bench number).

    TX_GEMM_STREAMK=0 python tools/step_ab.py mlp|logreg|lstm_small|lstm_medium [--steps K] [--reps R]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import paper_1605_02688_b200 as T
    from bench import time_device_block
    from oracle import configs as C
    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    if a.which in ("mlp", "logreg"):
        g = C.build_mlp(T) if a.which == "mlp" else C.build_logreg(T)
        f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
        host = C.inputs_mlp() if a.which == "mlp" else C.inputs_logreg()
    else:
        from tools.lstm_bench import CONFIGS, build
        H, L = CONFIGS[a.which.split("_")[1]]
        f, host = build(T, H, L)
    dev = [torch.from_numpy(v).cuda() for v in host]
    for _ in range(3):
        f.call_device(*dev)
    ms = [time_device_block(lambda: f.call_device(*dev), lib, f._stream, a.steps) for _ in range(a.reps)]
    env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("TX_"))
    print(f"{a.which} [{env or 'default'}]: median {statistics.median(ms) * 1e3:.1f} us/step, "
          f"min {min(ms) * 1e3:.1f} (reps {[round(x * 1e3, 1) for x in ms]})")


if __name__ == "__main__":
    main()
