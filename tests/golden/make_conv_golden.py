"""Convolution goldens from the REAL reference (texpr conv2d trio through
compile + grad): forward and both gradients for strided / padded float64 and
float32 cases.  Run in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_conv_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
CASES = [  # name, dtype, x shape, f shape, stride, pad, seed
    ("a", "float64", (2, 3, 9, 7), (4, 3, 3, 2), (2, 1), (1, 0), 1),
    ("b", "float64", (1, 2, 5, 5), (3, 2, 5, 5), (1, 1), (2, 2), 2),
    ("c", "float32", (4, 8, 16, 16), (16, 8, 3, 3), (1, 1), (1, 1), 3),
    ("d", "float32", (3, 5, 12, 10), (7, 5, 4, 3), (3, 2), (0, 1), 4),
]


def case_inputs(dtype, xs, fs, seed):
    r = np.random.default_rng(seed)
    x = r.standard_normal(xs).astype(dtype)
    f = (r.standard_normal(fs) * 0.3).astype(dtype)
    return x, f, r


def main():
    sys.path.insert(0, REF)
    import texpr as R
    out = {}
    for name, dt, xs, fs, st, pd, seed in CASES:
        x, f, r = case_inputs(dt, xs, fs, seed)
        vx, vf = R.tensor4("x", dtype=dt), R.tensor4("f", dtype=dt)
        y = R.conv2d(vx, vf, stride=st, pad=pd)
        fn0 = R.compile([vx, vf], [y])
        (yv,) = fn0(x, f)
        wgt = r.standard_normal(yv.shape).astype(dt)
        cost = R.sum(y * R.as_variable(wgt))
        gx, gf = R.grad(cost, [vx, vf])
        fn = R.compile([vx, vf], [y, gx, gf])
        for k, v in zip(("y", "gx", "gf"), fn(x, f)):
            out[f"{name}_{k}"] = v
        out[f"{name}_w"] = wgt
    np.savez(os.path.join(HERE, "ref_conv_goldens.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
