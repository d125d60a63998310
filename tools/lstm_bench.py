"""PTB-style LSTM language-model training step through ``scan`` (the paper's
LSTM benchmark shapes: batch 20; small 200 hidden x 20
steps, medium 600 x 40).  Synthetic embeddings and one-hot targets (no
dataset download), vocabulary 10000, softmax + cross-entropy per step inside
the loop, BPTT through ``grad``, SGD updates of every weight.  Reports words
per second (B x T words per step).

    python tools/lstm_bench.py [small|medium] [--steps K]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

CONFIGS = {"small": (200, 20), "medium": (600, 40)}


def build(T, H, L, B=20, V=10000, lr=0.1, seed=0, exclude=()):
    """``T`` is this package or the reference ``texpr`` (same spelling)."""
    import importlib
    ops = importlib.import_module(T.__name__ + ".ops")
    dimshuffle, subtensor = ops.dimshuffle, ops.subtensor
    rng = np.random.default_rng(seed)
    f32 = "float32"

    def sh(shape, scale, name):
        return T.shared((rng.standard_normal(shape) * scale).astype(np.float32), name=name)
    Wx, Wh = sh((H, 4 * H), 0.05, "Wx"), sh((H, 4 * H), 0.05, "Wh")
    bg = T.shared(np.zeros(4 * H, np.float32), name="bg")
    Wo, bo = sh((H, V), 0.05, "Wo"), T.shared(np.zeros(V, np.float32), name="bo")
    xs = T.tensor3("xs", dtype=f32)      # [L, B, H] embedded words
    ys = T.tensor3("ys", dtype=f32)      # [L, B, V] one-hot next words
    h0, c0 = T.matrix("h0", dtype=f32), T.matrix("c0", dtype=f32)

    def cell(x, y, h, c, wx, wh, b, wo, bo_):
        z = T.dot(x, wx) + T.dot(h, wh) + b
        i, f, o, g = (subtensor(z, (slice(None), slice(k * H, (k + 1) * H))) for k in range(4))
        c2 = T.sigmoid(f) * c + T.sigmoid(i) * T.tanh(g)
        h2 = T.sigmoid(o) * T.tanh(c2)
        logits = T.dot(h2, wo) + bo_
        m = T.max(logits, axis=1)
        e = T.exp(logits - dimshuffle(m, (0, "x")))
        p = e / dimshuffle(T.sum(e, axis=1), (0, "x"))
        return h2, c2, -T.sum(y * T.log(p))
    (_, _, costs), _ = T.scan(cell, sequences=[xs, ys], initial_states=[h0, c0],
                              non_sequences=[Wx, Wh, bg, Wo, bo])
    cost = T.sum(costs) / float(L * B)
    params = [Wx, Wh, bg, Wo, bo]
    grads = T.grad(cost, params)
    step = T.compile([xs, ys, h0, c0], [cost], updates=[(p, p - lr * g) for p, g in zip(params, grads)],
                     exclude=exclude)
    data_rng = np.random.default_rng(seed + 1)
    x = (data_rng.standard_normal((L, B, H)) * 0.5).astype(np.float32)
    y = np.eye(V, dtype=np.float32)[data_rng.integers(0, V, (L, B))]
    z = np.zeros((B, H), np.float32)
    return step, (x, y, z, z)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="medium")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch

    import paper_1605_02688_b200 as T
    from paper_1605_02688_b200 import native
    torch.cuda.set_device(0)
    lib = native.device_library(0)
    H, L = CONFIGS[a.config]
    t0 = time.perf_counter()
    step, host = build(T, H, L)
    dev = [torch.from_numpy(v).cuda() for v in host]
    c0 = float(step.call_device(*dev, sync=True)[0].item())
    t1 = time.perf_counter()
    for _ in range(3):
        step.call_device(*dev)
    e0, e1 = lib.event_create(), lib.event_create()
    lib.stream_sync(step._stream)
    lib.event_record(e0, step._stream)
    for _ in range(a.steps):
        step.call_device(*dev)
    lib.event_record(e1, step._stream)
    lib.stream_sync(step._stream)
    ms = lib.elapsed_ms(e0, e1) / a.steps
    c1 = float(step.call_device(*dev, sync=True)[0].item())
    plan = next(iter(step._plans.values()))
    nk = len(plan.launches) + sum(len(sp.launches) for sp in plan.subplans)
    print(f"lstm {a.config}: H={H} T={L} B=20 V=10000: {ms:.3f} ms/step, {20 * L / (ms * 1e-3):.0f} words/s, "
          f"cost {c0:.4f} -> {c1:.4f}, ~{nk} launches/step, first call (compile+plan) {t1 - t0:.1f} s")


if __name__ == "__main__":
    main()
