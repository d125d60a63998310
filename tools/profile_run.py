"""Short workload driver for ncu captures (never a bench number).

    python tools/profile_run.py [--only ew|mlp|logreg|reduce] [--steps N] [--gemm-mode auto|3xtf32|simt]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1605_02688_b200 as T  # noqa: E402
from oracle import configs as C  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--B", type=int, default=8192)
    ap.add_argument("--gemm-mode", default="auto")
    ap.add_argument("--dp", action="store_true", help="MLP through the data-parallel path (1 rank)")
    ap.add_argument("--n-global", type=int, default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    if a.only in ("all", "ew"):
        g = C.build_ew(T)
        f = T.compile(g["inputs"], g["outputs"])
        ins = [torch.randn(1 << 28, device="cuda") for _ in range(4)]
        for _ in range(a.steps):
            f.call_device(*ins, sync=True)
        del ins
    if a.only in ("all", "mlp"):
        g = C.build_mlp(T, B=a.B, n_global=a.n_global)
        dp = None
        if a.dp:
            from paper_1605_02688_b200.dp import DataParallel
            dp = DataParallel(world_size=1, rank=0)
        f = T.compile(g["inputs"], g["outputs"], updates=g["updates"], gemm_mode=a.gemm_mode, data_parallel=dp)
        x, y = C.inputs_mlp(B=a.B)
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        for _ in range(a.steps):
            f.call_device(xd, yd, sync=True)
        print("mlp nodes:", [getattr(n.op, "display_name", n.op.name) for n in f.order
                             if not getattr(n.op, "view_capable", False)])
    if a.only in ("all", "logreg"):
        g = C.build_logreg(T)
        f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
        x, y = C.inputs_logreg()
        xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        for _ in range(a.steps):
            f.call_device(xd, yd, sync=True)
        print("logreg nodes:", [getattr(n.op, "display_name", n.op.name) for n in f.order
                                if not getattr(n.op, "view_capable", False)])
    if a.only in ("all", "reduce"):
        X = torch.randn(16384, 16384, device="cuda")
        v = T.matrix("X", dtype="float32")
        for build in (T.sum, T.max, T.argmax):
            for ax in ((0,), (1,), None):
                f = T.compile([v], build(v, axis=ax))
                for _ in range(a.steps):
                    f.call_device(X, sync=True)
    torch.cuda.synchronize()
    print("done")


if __name__ == "__main__":
    main()
