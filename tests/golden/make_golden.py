"""Generate golden vectors by running the REAL reference (texpr) on seeded
inputs.  Run in the build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/texpr_goldens.npz (inputs are regenerated from the seeds
recorded here; only small inputs and all outputs are stored).  The GPU box
never runs this script; tests only read the .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "texpr_goldens.npz")


def main():
    sys.path.insert(0, REF)
    import texpr as T
    from texpr.graph import apply
    from texpr.ops import dimshuffle, make
    from texpr.ops.reductions import ArgmaxOnehot

    g = {"numpy_version": np.array(np.__version__)}
    rng = np.random.default_rng(2024)

    # ---- per-kernel elementwise goldens (preset none: plain Elemwise.perform)
    specials = np.array([0.0, -0.0, 1.0, -1.0, 0.5, -2.5, 3.0, 1e-30, -1e30, 88.0, -100.0, np.inf, -np.inf, np.nan],
                        dtype=np.float64)
    for dt in ("float32", "float64"):
        a = np.concatenate([specials, rng.standard_normal(50) * 3]).astype(dt)
        b = np.concatenate([specials[::-1], rng.standard_normal(50) * 3]).astype(dt)
        c = (rng.random(a.shape) > 0.5)
        g[f"ew_{dt}_a"], g[f"ew_{dt}_b"], g[f"ew_{dt}_c"] = a, b, c
        va, vb = T.vector("a", dtype=dt), T.vector("b", dtype=dt)
        vc = T.vector("c", dtype="bool")
        for k in ("add", "sub", "mul", "div", "pow", "maximum", "lt", "gt", "le", "ge", "eq", "neq", "second"):
            f = T.compile([va, vb], make(k, [va, vb]), preset="none")
            g[f"ew_{dt}_{k}"] = f(a, b)
        for k in ("neg", "exp", "log", "log1p", "sqr", "sqrt", "sigmoid", "tanh", "isnan"):
            f = T.compile([va], make(k, [va]), preset="none")
            g[f"ew_{dt}_{k}"] = f(a)
        f = T.compile([vc, va, vb], make("switch", [vc, va, vb]), preset="none")
        g[f"ew_{dt}_switch"] = f(c, a, b)
    # integer kernels
    ia = rng.integers(-50, 50, 64).astype(np.int64)
    ib = rng.integers(1, 9, 64).astype(np.int64) * np.where(rng.random(64) > 0.5, 1, -1)
    g["ew_int64_a"], g["ew_int64_b"] = ia, ib
    va, vb = T.vector("a", dtype="int64"), T.vector("b", dtype="int64")
    for k in ("add", "sub", "mul", "div", "maximum", "lt", "eq"):
        g[f"ew_int64_{k}"] = T.compile([va, vb], make(k, [va, vb]), preset="none")(ia, ib)

    # ---- broadcasting elementwise: bias row + column
    X = rng.standard_normal((17, 23)).astype(np.float32)
    r = rng.standard_normal(23).astype(np.float32)
    col = rng.standard_normal((17, 1)).astype(np.float32)
    g["bc_X"], g["bc_r"], g["bc_col"] = X, r, col
    vX = T.matrix("X", dtype="float32")
    vr = T.vector("r", dtype="float32")
    vcol = T.matrix("col", dtype="float32", broadcastable=(False, True))
    g["bc_out"] = T.compile([vX, vr, vcol], T.tanh(vX + vr) * vcol - vr, preset="fast_run")(X, r, col)

    # ---- reductions, incl. ties and NaN
    R = rng.standard_normal((37, 53)).astype(np.float32)
    R[3, :] = 1.5           # full-row tie -> first index
    R[:, 7] = 2.5           # full-column tie
    R[5, 11] = np.nan       # NaN wins argmax, propagates in max
    R[20, 40] = np.nan
    R[21, 40] = np.nan
    g["red_X"] = R
    vR = T.matrix("R", dtype="float32")
    for ax in ((0,), (1,), (0, 1)):
        tag = "".join(map(str, ax))
        g[f"red_sum_{tag}"] = T.compile([vR], T.sum(vR, axis=ax), preset="fast_run")(R)
        g[f"red_max_{tag}"] = T.compile([vR], T.max(vR, axis=ax), preset="fast_run")(R)
        g[f"red_argmax_onehot_{tag}"] = T.compile([vR], apply(ArgmaxOnehot(ax), [vR])[0])(R)
    R3 = rng.standard_normal((5, 6, 7)).astype(np.float64)
    g["red3_X"] = R3
    v3 = T.tensor3("R3", dtype="float64")
    for ax in ((0, 2), (1,), (0, 1, 2), (2,), (0,)):
        tag = "".join(map(str, ax))
        g[f"red3_sum_{tag}"] = T.compile([v3], T.sum(v3, axis=ax))(R3)
        g[f"red3_max_{tag}"] = T.compile([v3], T.max(v3, axis=ax))(R3)
        g[f"red3_argmax_onehot_{tag}"] = T.compile([v3], apply(ArgmaxOnehot(ax), [v3])[0])(R3)

    # ---- dot variants
    A = rng.standard_normal((33, 17)).astype(np.float32)
    Bm = rng.standard_normal((17, 29)).astype(np.float32)
    v = rng.standard_normal(17).astype(np.float32)
    g["dot_A"], g["dot_B"], g["dot_v"] = A, Bm, v
    vA, vB, vv = T.matrix("A", dtype="float32"), T.matrix("B", dtype="float32"), T.vector("v", dtype="float32")
    g["dot_mm"] = T.compile([vA, vB], T.dot(vA, vB))(A, Bm)
    g["dot_mv"] = T.compile([vA, vv], T.dot(vA, vv))(A, v)
    g["dot_vm"] = T.compile([vv, vB], T.dot(vv, vB))(v, Bm)
    g["dot_vv"] = T.compile([vv], T.dot(vv, vv))(v)
    g["dot_tn"] = T.compile([vA], T.dot(T.transpose(vA), vA))(A)

    # ---- config 2 expression, fused (fast_run) and unfused (none)
    n = 40000
    r7 = np.random.default_rng(7)
    ew = [r7.standard_normal(n, dtype=np.float32) for _ in range(4)]
    a, b, c, d = (T.vector(s, dtype="float32") for s in "abcd")
    expr = T.sigmoid(a * b + c) ** 2 - d
    g["cfg2_fused"] = T.compile([a, b, c, d], expr, preset="fast_run")(*ew)
    g["cfg2_unfused"] = T.compile([a, b, c, d], expr, preset="none")(*ew)

    # ---- config 1: two logreg SGD steps (full size; inputs from seed 0)
    def sxent(z, y, n_):
        m = T.max(z, axis=1)
        e = T.exp(z - dimshuffle(m, (0, "x")))
        p = e / dimshuffle(T.sum(e, axis=1), (0, "x"))
        return -T.sum(y * T.log(p)) / float(n_)

    r0 = np.random.default_rng(0)
    x = r0.random((600, 784), dtype=np.float32)
    y = np.eye(10, dtype=np.float32)[r0.integers(0, 10, 600)]
    vx, vy = T.matrix("x", dtype="float32"), T.matrix("y", dtype="float32")
    W = T.shared(np.zeros((784, 10), np.float32), name="W")
    bb = T.shared(np.zeros(10, np.float32), name="b")
    cost = sxent(T.dot(vx, W) + bb, vy, 600)
    gW, gb = T.grad(cost, [W, bb])
    step = T.compile([vx, vy], [cost], updates=[(W, W - 0.13 * gW), (bb, bb - 0.13 * gb)],
                     preset="fast_run", exclude=("fuse_elemwise",))
    costs = [step(x, y)[0] for _ in range(3)]
    g["cfg1_costs"] = np.array(costs)
    g["cfg1_W"] = W.get_value()
    g["cfg1_b"] = bb.get_value()
    g["cfg1_nodes"] = np.array(len(step.order))

    # ---- config 4 at reduced size (B=64, H=96): two MLP SGD steps
    B, D, H, K = 64, 784, 96, 10
    rr = np.random.default_rng(0)
    Ws = [(rr.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32) for i, o in ((D, H), (H, H), (H, K))]
    r1 = np.random.default_rng(1)
    xm = r1.random((B, D), dtype=np.float32)
    ym = np.eye(K, dtype=np.float32)[r1.integers(0, K, B)]
    W1, W2, W3 = (T.shared(w, name=f"W{i}") for i, w in enumerate(Ws))
    b1, b2, b3 = (T.shared(np.zeros(k, np.float32), name=f"b{k}") for k in (H, H, K))
    h1 = T.tanh(T.dot(vx, W1) + b1)
    h2 = T.tanh(T.dot(h1, W2) + b2)
    cost = sxent(T.dot(h2, W3) + b3, vy, B)
    params = [W1, b1, W2, b2, W3, b3]
    grads = T.grad(cost, params)
    step = T.compile([vx, vy], [cost], updates=[(p, p - 0.01 * gr) for p, gr in zip(params, grads)],
                     preset="fast_run", exclude=("fuse_elemwise",))
    g["cfg4_costs"] = np.array([step(xm, ym)[0] for _ in range(2)])
    for i, p in enumerate(params):
        g[f"cfg4_p{i}"] = p.get_value()
    g["cfg4_nodes"] = np.array(len(step.order))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays")


if __name__ == "__main__":
    main()
