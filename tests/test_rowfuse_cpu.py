"""Row fusion on CPU: with concrete shapes, the logistic-regression step's
softmax / cross-entropy block (forward, grad, bias-gradient and cost batch
sums) forms one convex group, and the generated kernel compiles with NVRTC
for sm_100a (compile only; execution is covered by the GPU tests)."""
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C
from paper_1605_02688_b200 import native, rowfuse


class _Lay:
    def __init__(self, shape):
        self.shape = tuple(shape)


class _FakePlan:
    """Just the shape map the grouping and codegen read."""

    def __init__(self, fg, in_shapes):
        self.lay = {}
        for v, s in zip(fg.inputs, in_shapes):
            self.lay[v.id] = _Lay(s)
        for n in fg.toposort():
            shp = [self.lay[x.id].shape if x.id in self.lay else x.value.shape for x in n.inputs]
            for o, s in zip(n.outputs, n.op.infer_shape(n, shp)):
                self.lay[o.id] = _Lay(s)


def _shapes(f, in_shapes):
    """Input shapes in fg.inputs order: explicit inputs, then shared values."""
    return list(in_shapes) + [f.values[id(s)].shape for s in f.shared]


def _logreg(N=600):
    g = C.build_logreg(T, N=N)
    f = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"])
    return f.fg, _FakePlan(f.fg, _shapes(f, [(N, 784), (N, 10)]))


def test_logreg_softmax_block_is_one_group():
    fg, plan = _logreg()
    order = fg.toposort()
    groups = rowfuse.find_groups(plan, order, fg)
    assert len(groups) == 1
    grp = groups[0]
    kinds = [getattr(n.op, "display_name", n.op.name) for n in grp.launchable()]
    # everything between the logits GEMM and dW = x^T dz is in the group,
    # including the cost's sum[0,1] and the bias gradient's sum[0] (sinks)
    assert "dot" not in kinds
    assert "sum[0, 1]" in kinds and "sum[0]" in kinds and "max[1]" in kinds
    outside = [n for n in order if n.id not in grp.member_ids and not getattr(n.op, "view_capable", False)]
    assert len(outside) <= 6


def test_generated_row_kernel_compiles():
    fg, plan = _logreg()
    grp = rowfuse.find_groups(plan, fg.toposort(), fg)[0]
    gen = rowfuse._Gen(grp, plan, fg)
    for n in grp.members:
        gen.node(n)
    store = {}
    for n in grp.members:
        for o in n.outputs:
            if o.id not in grp.sink_vars and (fg.is_output(o) or any(c.id not in grp.member_ids for c in fg.node_clients(o))):
                store[o.id] = o
    gen.stores(store)
    total = gen.finish_sinks()
    src = gen.source(gen.lines, total)
    assert native.library().ew_check(src, "rowcheck") > 0
    assert total == 10 + 1  # db (10 columns) + cost sum


def test_wide_rows_do_not_group():
    g = C.build_mlp(T, B=64, H=512)
    f = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"])
    plan = _FakePlan(f.fg, _shapes(f, [(64, 784), (64, 10)]))
    groups = rowfuse.find_groups(plan, f.fg.toposort(), f.fg)
    for grp in groups:
        assert grp.K == 10  # only the softmax layer's [B,10] block fuses
