"""Loop goldens from the REAL reference (texpr scan, float64): an RNN's
histories, final state, BPTT gradients and R-operator, a nested loop, and a
last-step-only loop after the reference's fast_run loop rewrites.  Run in the
build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_scan_golden.py

Inputs are regenerated from the seeds below by tests/test_device_scan.py.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def rnn_point(seed=7, length=9, size=5):
    r = np.random.default_rng(seed)
    return [r.standard_normal((length, size)) * 0.5, r.standard_normal(size) * 0.5,
            r.standard_normal((size, size)) * 0.4, r.standard_normal((size, size)) * 0.4,
            r.standard_normal((length, size)), r.standard_normal(size),
            r.standard_normal((size, size)), r.standard_normal((size, size))]


def main():
    sys.path.insert(0, REF)
    import texpr as R
    from texpr.scan import scan
    out = {}
    xs, h0, w, u = R.matrix("xs"), R.vector("h0"), R.matrix("w"), R.matrix("u")
    dirs = [R.matrix("dxs"), R.vector("dh0"), R.matrix("dw"), R.matrix("du")]

    def step(x_t, h_prev, w_, u_):
        return R.tanh(R.dot(w_, h_prev) + R.dot(u_, x_t))
    (hist,), (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    cost = R.sum(R.sqr(final)) + R.sum(hist * 0.5)
    grads = R.grad(cost, [xs, h0, w, u])
    jv = R.rop([final], [xs, h0, w, u], dirs)[0]
    f = R.compile([xs, h0, w, u] + dirs, [hist, final] + grads + [jv])
    vals = f(*rnn_point())
    for k, v in zip(["rnn_hist", "rnn_final", "rnn_gxs", "rnn_gh0", "rnn_gw", "rnn_gu", "rnn_rop"], vals):
        out[k] = v

    xv, a0 = R.vector("xv"), R.scalar("a0")

    def outer_step(x_t, acc):
        _, (inner_final,) = scan(lambda s, x: R.tanh(s + x), initial_states=[acc], non_sequences=[x_t], n_steps=3)
        return acc * 0.5 + inner_final
    (nh,), (nf,) = scan(outer_step, sequences=[xv], initial_states=[a0])
    gn = R.grad(nf, [xv, a0])
    fn = R.compile([xv, a0], [nh, nf] + gn)
    r = np.random.default_rng(11)
    vals = fn(r.standard_normal(6) * 0.5, np.array(0.2))
    for k, v in zip(["nest_hist", "nest_final", "nest_gx", "nest_ga"], vals):
        out[k] = v

    ys = R.vector("ys")
    (lh,), _ = scan(lambda x, s: s * 0.9 + R.tanh(x), sequences=[ys], initial_states=[R.as_variable(0.0)])
    fl = R.compile([ys], [lh[-1] * 2.0], preset="fast_run")
    out["last_out"] = fl(np.random.default_rng(13).standard_normal(40))[0]
    np.savez(os.path.join(HERE, "ref_scan_goldens.npz"), **out)
    print({k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
