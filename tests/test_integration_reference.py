"""The boundary from the other side: the UNMODIFIED reference runtime (texpr
from baseline/_ref) with the B200 library plugged in through the reference's
own plugin API (integration/texpr_b200.py: ``@register_op`` + an
``abstract_select`` rewrite routing Dot to ``tx_gemm``), versus the same
reference program on its CPU path.  INTEGRATION.md §2, executed.

Skipped when the reference is not installed in baseline/_ref (git-ignored;
made by ``pip install --target baseline/_ref``)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
LIB = os.path.join(ROOT, "paper_1605_02688_b200", "libtexpr_b200.so")


@pytest.fixture(scope="module")
def texpr_b200():
    if not os.path.isdir(os.path.join(REF, "texpr")):
        pytest.skip("reference not installed in baseline/_ref")
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import texpr
    import texpr_b200
    lib, op = texpr_b200.install(texpr, LIB, precision="3xtf32")
    return texpr, lib, op


def _mlp(texpr, B, H, seed=0):
    from texpr.ops import dimshuffle
    rng = np.random.default_rng(seed)
    f32 = "float32"

    def wsh(i, o, n):
        return texpr.shared((rng.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32), name=n)
    x, y = texpr.matrix("x", dtype=f32), texpr.matrix("y", dtype=f32)
    W1, W2, W3 = wsh(784, H, "W1"), wsh(H, H, "W2"), wsh(H, 10, "W3")
    b1, b2, b3 = (texpr.shared(np.zeros(k, np.float32), name=n) for k, n in ((H, "b1"), (H, "b2"), (10, "b3")))
    h1 = texpr.tanh(texpr.dot(x, W1) + b1)
    h2 = texpr.tanh(texpr.dot(h1, W2) + b2)
    z = texpr.dot(h2, W3) + b3
    m = texpr.max(z, axis=1)
    e = texpr.exp(z - dimshuffle(m, (0, "x")))
    p = e / dimshuffle(texpr.sum(e, axis=1), (0, "x"))
    cost = -texpr.sum(y * texpr.log(p)) / float(B)
    params = [W1, b1, W2, b2, W3, b3]
    grads = texpr.grad(cost, params)
    return [x, y], [cost], [(q, q - 0.01 * g) for q, g in zip(params, grads)], params


def test_reference_runtime_runs_dot_on_b200(texpr_b200):
    texpr, lib, B200Dot = texpr_b200
    B, H = 256, 512
    r = np.random.default_rng(1)
    xv = r.random((B, 784), dtype=np.float32)
    yv = np.eye(10, dtype=np.float32)[r.integers(0, 10, B)]
    ins, outs, ups, pa = _mlp(texpr, B, H)
    cpu = texpr.compile(ins, outs, updates=ups, preset="fast_run", exclude=("fuse_elemwise",))
    ins2, outs2, ups2, pb = _mlp(texpr, B, H)
    dev = texpr.compile(ins2, outs2, updates=ups2, preset="fast_run", exclude=("fuse_elemwise",),
                        include=("b200_select_dot",))
    names = [n.op.name for n in dev.order]
    assert names.count("b200_dot") == 8 and "dot" not in names, names
    assert [n.op.name for n in cpu.order].count("dot") == 8
    before = lib.calls
    for _ in range(3):
        c_cpu, c_dev = float(cpu(xv, yv)[0]), float(dev(xv, yv)[0])
        assert abs(c_dev - c_cpu) <= 1e-5 * abs(c_cpu), (c_dev, c_cpu)
    assert lib.calls - before == 3 * 8
    for q, s in zip(pa, pb):
        a, b = q.get_value().astype(np.float64), s.get_value().astype(np.float64)
        assert np.linalg.norm(a - b) <= 1e-5 * max(np.linalg.norm(a), 1e-30), q.name
