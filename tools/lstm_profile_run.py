"""LSTM step driver for ncu launch lists (never a bench number).

    python tools/lstm_profile_run.py [small|medium] [--calls N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="small")
    ap.add_argument("--calls", type=int, default=2)
    a = ap.parse_args()
    import torch

    import paper_1605_02688_b200 as T
    from tools.lstm_bench import CONFIGS, build
    torch.cuda.set_device(0)
    H, L = CONFIGS[a.config]
    step, host = build(T, H, L)
    dev = [torch.from_numpy(v).cuda() for v in host]
    for _ in range(a.calls):
        step.call_device(*dev, sync=True)
    inner = [n for n in step.order if n.op.name == "scan"]
    for n in inner:
        fn = n.op._inner_fn
        if fn is not None:
            print(n.op.display_name, "body:", [getattr(m.op, "display_name", m.op.name) for m in fn.order
                                               if not getattr(m.op, "view_capable", False)])
    print("outer:", [getattr(m.op, "display_name", m.op.name) for m in step.order
                     if not getattr(m.op, "view_capable", False)])


if __name__ == "__main__":
    main()
