"""Per-launch device times of one compiled step, grouped by node (diagnostic,
never a bench number): every launch of the top plan and of each unrolled
scan body is timed alone between two events on the VM stream.

    python tools/plan_profile.py lstm_small|lstm_medium|mlp [--top 25]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("work")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    import torch
    import paper_1605_02688_b200 as T
    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    if a.work.startswith("lstm"):
        from tools.lstm_bench import CONFIGS, build
        H, L = CONFIGS[a.work.split("_")[1]]
        step, host = build(T, H, L)
        dev = [torch.from_numpy(v).cuda() for v in host]
    else:
        from oracle import configs as C
        g = C.build_mlp(T, B=8192)
        step = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
        x, y = C.inputs_mlp(B=8192)
        dev = [torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()]
    for _ in range(3):
        step.call_device(*dev, sync=True)
    plan = next(iter(step._plans.values()))
    st = step._stream
    e0, e1 = lib.event_create(), lib.event_create()
    agg = collections.defaultdict(lambda: [0, 0.0])

    def label(node, owner):
        if node is None:
            return "copy/fill (no node)"
        op = node.op
        nm = type(op).__name__
        k = getattr(op, "kernel", None) or getattr(op, "name", None)
        shapes = []
        for v in node.outputs[:1]:
            try:
                shapes.append(tuple(owner.lay[v.id].shape))
            except Exception:
                shapes.append("?")
        return f"{nm}{'[' + str(k) + ']' if isinstance(k, str) else ''} {shapes}"

    def run_list(launches, sub, owner):
        for node, fn in launches:
            lib.stream_sync(st)
            lib.event_record(e0, st)
            fn(st)
            lib.event_record(e1, st)
            lib.stream_sync(st)
            lab = ("body: " if sub else "") + (label(node, owner) if node is not None else "copy/fill")
            r = agg[lab]
            r[0] += 1
            r[1] += lib.elapsed_ms(e0, e1) * 1e3
    # the top plan's launches include the scan launcher (which runs every body);
    # time the bodies separately and the top plan's own launches
    for sp in plan.subplans:
        run_list(sp.launches, True, sp)
    for node, fn in plan.launches:
        if node is not None and type(node.op).__name__ == "ScanOp":
            continue
        run_list([(node, fn)], False, plan)
    tot = sum(v[1] for v in agg.values())
    print(f"{a.work}: {tot:.1f} us summed over {sum(v[0] for v in agg.values())} launches (each timed alone)")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:a.top]:
        print(f"  {t:8.1f} us  {n:4d} x {t / n:6.2f}  {k}")


if __name__ == "__main__":
    main()
