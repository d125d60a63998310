"""Function-container (TXFN v1) fixtures made by the REAL reference, and a
cross-check that the reference loads what this package saves.  Run in the
build container, where /root/reference exists:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_txfn.py

Writes (committed; the GPU box only reads them):
  ref_logreg_after2.txfn   reference logreg step (config 1 recipe, N=600,
                           fast_run - fuse_elemwise) saved after 2 SGD steps
  ref_ew.txfn              reference fast_run composite sigmoid(a*b+c)**2-d
  ref_txfn_expect.npz      what the reference computes next: the 3rd logreg
                           step (cost, W, b) and the EW outputs on seed-5 data
It also asserts that a container saved by THIS package (portable graph) loads
in the reference and reproduces the reference's own 3-step trajectory
bit-for-bit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"


def ref_logreg(R, lr=0.13, N=600):
    from texpr.ops import dimshuffle
    x, y = R.matrix("x", dtype="float32"), R.matrix("y", dtype="float32")
    W = R.shared(np.zeros((784, 10), np.float32), name="W")
    b = R.shared(np.zeros(10, np.float32), name="b")
    z = R.dot(x, W) + b
    m = R.max(z, axis=1)
    e = R.exp(z - dimshuffle(m, (0, "x")))
    p = e / dimshuffle(R.sum(e, axis=1), (0, "x"))
    cost = -R.sum(y * R.log(p)) / float(N)
    gW, gb = R.grad(cost, [W, b])
    f = R.compile([x, y], [cost], updates=[(W, W - lr * gW), (b, b - lr * gb)],
                  preset="fast_run", exclude=("fuse_elemwise",))
    return f, W, b


def main():
    sys.path.insert(0, ROOT)
    from oracle import configs as C
    x, y = C.inputs_logreg(N=600)

    # ---- containers written by THIS package (before the reference is imported)
    import paper_1605_02688_b200 as T
    g = C.build_logreg(T)
    ours = T.compile(g["inputs"], g["outputs"], updates=g["updates"]).save()
    gew = C.build_ew(T)
    ours_ew = T.compile(gew["inputs"], gew["outputs"]).save()

    sys.path.insert(0, REF)
    import texpr as R
    out = {}
    f, W, b = ref_logreg(R)
    costs = [float(f(x, y)[0]) for _ in range(2)]
    blob = R.save(f)
    open(os.path.join(HERE, "ref_logreg_after2.txfn"), "wb").write(blob)
    costs.append(float(f(x, y)[0]))
    out["logreg_costs"] = np.array(costs, np.float32)
    out["logreg_W3"], out["logreg_b3"] = W.get_value(), b.get_value()

    a, bb, c, d = (R.vector(s, dtype="float32") for s in "abcd")
    fe = R.compile([a, bb, c, d], R.sigmoid(a * bb + c) ** 2 - d, preset="fast_run")
    open(os.path.join(HERE, "ref_ew.txfn"), "wb").write(R.save(fe))
    ins = C.inputs_ew(1000, seed=5)
    out["ew_out"] = fe(*ins)

    # ---- the reference runs what this package saved: same trajectory, bit for bit
    g2 = R.load(ours)
    mine = [float(g2(x, y)[0]) for _ in range(3)]
    assert mine == costs, (mine, costs)
    ws = {s.name: s.get_value() for s, _ in g2.shared_bindings}
    assert np.array_equal(ws["W"], out["logreg_W3"]) and np.array_equal(ws["b"], out["logreg_b3"])
    e2 = R.load(ours_ew)
    assert np.array_equal(e2(*ins), out["ew_out"])
    print("reference loads this package's containers: logreg 3-step costs", mine, "(bit-exact), ew bit-exact")
    np.savez(os.path.join(HERE, "ref_txfn_expect.npz"), **out)


if __name__ == "__main__":
    main()
