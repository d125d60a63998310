"""The reference's own CPU path timed beside the GPU.

Runs the UNMODIFIED reference package (``texpr``, installed once into
``baseline/_ref`` with pip; git-ignored, travels to the GPU box) through its
public API -- ``texpr.compile(...)`` then ``f(*host_arrays)`` -- on the
SURVEY Appendix A recipes of the five BASELINE configs, at full size, on the
box's host cores:

  * ``e2e``: wall time of ``f(*values)`` (includes the reference's input copy,
    ``runtime.py:163-171``, and output copy, ``:412-417``);
  * ``kernel``: the sum of ``Profile.node_time`` for that call
    (``runtime.py:113-160``, ``:353-358``) -- the per-node perform() time only.

One warm-up call, then the median of ``reps`` calls.  Presets follow SURVEY
§8(c): ``fast_run`` for configs 2 and 3, ``fast_run`` minus ``fuse_elemwise``
for the training steps (plain ``fast_run`` raises CycleDetected there, F2).
"argmax" in the reference is ``ArgmaxOnehot`` (``ops/reductions.py:149-188``,
one-hot output of the input's shape): it is timed as such.

If ``baseline/_ref`` is missing the table is not produced (the caller falls
back to the oracle port for the headline reference arm).
"""
from __future__ import annotations

import os
import platform
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
F32 = "float32"


def load_reference():
    """The installed reference package, or None."""
    if not os.path.isdir(os.path.join(REF, "texpr")):
        return None
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import texpr
    if not os.path.abspath(texpr.__file__).startswith(REF):
        raise RuntimeError(f"texpr resolved to {texpr.__file__}, not baseline/_ref")
    return texpr


def host_info():
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads"), "version": i.get("version")}
                for i in threadpool_info()]
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model, "blas": blas,
            "numpy": np.__version__, "elementwise_threads": 1,
            "note": "NumPy ufuncs / reductions are single-threaded; only Dot (OpenBLAS sgemm) uses all cores"}


def _time(f, args, reps):
    """(median e2e s, median kernel-only s) over ``reps`` calls after 1 warm-up."""
    f(*args)
    e2e, kern = [], []
    for _ in range(reps):
        before = sum(f.profile.node_time.values())
        t0 = time.perf_counter()
        f(*args)
        e2e.append(time.perf_counter() - t0)
        kern.append(sum(f.profile.node_time.values()) - before)
    return statistics.median(e2e), statistics.median(kern)


def _xent(tx, z, y, n_global):
    from texpr.ops import dimshuffle
    m = tx.max(z, axis=1)
    e = tx.exp(z - dimshuffle(m, (0, "x")))
    p = e / dimshuffle(tx.sum(e, axis=1), (0, "x"))
    return -tx.sum(y * tx.log(p)) / float(n_global)


def _mlp(tx, B, n_global, H=4096, D=784, K=10, lr=0.01):
    rng = np.random.default_rng(0)

    def wsh(i, o, n):
        return tx.shared((rng.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32), name=n)
    x, y = tx.matrix("x", dtype=F32), tx.matrix("y", dtype=F32)
    W1, W2, W3 = wsh(D, H, "W1"), wsh(H, H, "W2"), wsh(H, K, "W3")
    b1, b2, b3 = (tx.shared(np.zeros(k, np.float32), name=n) for k, n in ((H, "b1"), (H, "b2"), (K, "b3")))
    h1 = tx.tanh(tx.dot(x, W1) + b1)
    h2 = tx.tanh(tx.dot(h1, W2) + b2)
    cost = _xent(tx, tx.dot(h2, W3) + b3, y, n_global)
    params = [W1, b1, W2, b2, W3, b3]
    grads = tx.grad(cost, params)
    f = tx.compile([x, y], [cost], updates=[(p, p - lr * g) for p, g in zip(params, grads)],
                   preset="fast_run", exclude=("fuse_elemwise",))
    r = np.random.default_rng(1)
    xv = r.random((B, D), dtype=np.float32)
    yv = np.eye(K, dtype=np.float32)[r.integers(0, K, B)]
    return f, (xv, yv)


def config1(tx, reps):
    x, y = tx.matrix("x", dtype=F32), tx.matrix("y", dtype=F32)
    W = tx.shared(np.zeros((784, 10), np.float32), name="W")
    b = tx.shared(np.zeros(10, np.float32), name="b")
    cost = _xent(tx, tx.dot(x, W) + b, y, 600)
    gW, gb = tx.grad(cost, [W, b])
    f = tx.compile([x, y], [cost], updates=[(W, W - 0.13 * gW), (b, b - 0.13 * gb)],
                   preset="fast_run", exclude=("fuse_elemwise",))
    r = np.random.default_rng(0)
    xv = r.random((600, 784), dtype=np.float32)
    yv = np.eye(10, dtype=np.float32)[r.integers(0, 10, 600)]
    e2e, k = _time(f, (xv, yv), reps * 20)
    return {"unit": "samples/s", "e2e": 600 / e2e, "kernel": 600 / k, "e2e_us_per_step": e2e * 1e6,
            "kernel_us_per_step": k * 1e6, "nodes": len(f.order)}


def config2(tx, reps, n=1 << 28):
    a, bb, c, d = (tx.vector(s, dtype=F32) for s in "abcd")
    f = tx.compile([a, bb, c, d], tx.sigmoid(a * bb + c) ** 2 - d, preset="fast_run")
    r = np.random.default_rng(0)
    ins = [r.standard_normal(n, dtype=np.float32) for _ in range(4)]
    e2e, k = _time(f, ins, reps)
    return {"unit": "GB/s", "e2e": 20 * n / e2e / 1e9, "kernel": 20 * n / k / 1e9, "e2e_s": e2e, "kernel_s": k,
            "elements": n, "nodes": len(f.order)}


def config3(tx, reps, n=16384):
    from texpr.graph import apply
    from texpr.ops.reductions import ArgmaxOnehot
    X = tx.matrix("X", dtype=F32)
    Xv = np.random.default_rng(0).standard_normal((n, n), dtype=np.float32)
    out = {"unit": "GB/s (input bytes read)"}
    for kind in ("sum", "max", "argmax_onehot"):
        for ax, tag in (((0,), "axis0"), ((1,), "axis1"), (None, "all")):
            if kind == "argmax_onehot":
                expr = apply(ArgmaxOnehot((0, 1) if ax is None else ax), [X])[0]
            else:
                expr = (tx.sum if kind == "sum" else tx.max)(X, axis=None if ax is None else ax[0])
            f = tx.compile([X], expr, preset="fast_run")
            e2e, k = _time(f, (Xv,), reps)
            out[f"{kind}_{tag}"] = {"e2e": n * n * 4 / e2e / 1e9, "kernel": n * n * 4 / k / 1e9,
                                    "e2e_s": e2e, "kernel_s": k}
    return out


def config4(tx, reps, B=8192):
    f, args = _mlp(tx, B, B)
    e2e, k = _time(f, args, reps)
    return {"unit": "samples/s", "e2e": B / e2e, "kernel": B / k, "e2e_s": e2e, "kernel_s": k, "batch": B,
            "nodes": len(f.order)}


def config5(tx, reps, G=65536):
    f, args = _mlp(tx, G, G)
    e2e, k = _time(f, args, reps)
    return {"unit": "samples/s", "e2e": G / e2e, "kernel": G / k, "e2e_s": e2e, "kernel_s": k,
            "global_batch": G, "processes": 1, "note": "the reference has no data parallelism: one process"}


CONV = dict(N=32, C=64, H=56, W=56, K=64, kh=3, kw=3, pad=(1, 1))


def conv_graph(tx, shared_value, lr=1e-3):
    """A 3x3 convolution layer's training step (SURVEY §8(f)3 shapes: a
    ResNet conv2_x layer): forward, both gradients, SGD on the filters.
    ``tx`` is either package (same spelling)."""
    d = CONV
    x = tx.tensor4("x", dtype=F32)
    f = tx.shared(shared_value, name="f")
    y = tx.conv2d(x, f, stride=(1, 1), pad=d["pad"])
    cost = tx.sum(y * y) * 1e-6
    gf, gx = tx.grad(cost, [f, x])
    return [x], [cost, gx], [(f, f - lr * gf)]


def conv_inputs():
    d = CONV
    r = np.random.default_rng(7)
    x = r.standard_normal((d["N"], d["C"], d["H"], d["W"]), dtype=np.float32)
    f = (r.standard_normal((d["K"], d["C"], d["kh"], d["kw"])) / np.sqrt(d["C"] * 9)).astype(np.float32)
    return x, f


CONV_FLOP = 3 * 2 * CONV["N"] * CONV["K"] * CONV["C"] * CONV["kh"] * CONV["kw"] * CONV["H"] * CONV["W"]


def config_conv(tx, reps):
    x, f0 = conv_inputs()
    ins, outs, ups = conv_graph(tx, f0)
    f = tx.compile(ins, outs, updates=ups, preset="fast_run", conv_impl="gemm")
    e2e, k = _time(f, (x,), reps)
    return {"unit": "TFLOP/s (fwd + grad_w + grad_x)", "e2e": CONV_FLOP / e2e / 1e12, "kernel": CONV_FLOP / k / 1e12,
            "e2e_s": e2e, "kernel_s": k, "shape": dict(CONV)}


def config_lstm(tx, reps):
    """The PTB LSTM language-model step (tools/lstm_bench.py: scan over T steps,
    softmax-xent per step, BPTT, SGD) on the reference's CPU path."""
    from tools.lstm_bench import CONFIGS, build
    out = {"unit": "words/s"}
    for name, (H, L) in CONFIGS.items():
        f, args = build(tx, H, L, exclude=("fuse_elemwise",))
        e2e, k = _time(f, args, max(2, reps // 2))
        out[name] = {"e2e": 20 * L / e2e, "kernel": 20 * L / k, "e2e_s": e2e, "kernel_s": k, "hidden": H, "steps": L}
    return out


def table(reps=5, only=None):
    """Every config's CPU-path throughput (end-to-end and kernel-only)."""
    tx = load_reference()
    if tx is None:
        return None
    res = {"kind": "reference", "source": "baseline/_ref texpr (unmodified, pip-installed from /root/reference)",
           "calls": f"1 warm-up + median of {reps}", "host": host_info()}
    for name, fn in (("config1_logreg_n600", config1), ("config2_ew_2p28", config2),
                     ("config3_careduce_16384sq", config3), ("config4_mlp_b8192", config4),
                     ("config5_mlp_global65536", config5), ("conv3x3_n32c64h56", config_conv),
                     ("lstm_ptb", config_lstm)):
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        try:
            res[name] = _round(fn(tx, reps))
        except Exception as e:  # pragma: no cover - reported, not hidden
            res[name] = {"error": repr(e)[:300]}
        res[name]["wall_s"] = round(time.perf_counter() - t0, 1)
    return res


def _round(d):
    if isinstance(d, dict):
        return {k: _round(v) for k, v in d.items()}
    if isinstance(d, float):
        return float(f"{d:.5g}")
    return d


if __name__ == "__main__":
    import json
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    print(json.dumps(table(reps, only)))
