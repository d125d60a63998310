"""Builder namespace (reference ``texpr.ops``, ``ops/__init__.py:83-137``).

``from paper_1605_02688_b200.ops import dimshuffle`` and friends resolve here,
so reference programs port by changing the import line only.
"""
from __future__ import annotations

from .elemwise import (KERNELS, Composite, CompositeElemwise, Elemwise, fill, make,  # noqa: F401
                       ones_like, sum_to_matching_shape, zeros_like)
from .graph import Variable
from .linalg import Dot, dot  # noqa: F401
from .op import DISCONNECTED, OP_REGISTRY, UNKNOWN_SHAPE, Op, op_from_payload, register_op  # noqa: F401
from .reduce import Argmax, ArgmaxOnehot, Max, Sum, argmax, argmax_onehot, max, sum  # noqa: F401
from .shaping import (DimShuffle, IncSubtensor, Join, Reshape, ShapeOf, Subtensor, dimshuffle, flip0,  # noqa: F401
                      inc_subtensor, join, reshape, shape_of, subtensor, transpose)
from .conv import Conv2d, conv2d  # noqa: F401


def _binary(kernel):
    def build(a, b):
        return make(kernel, [a, b])
    build.__name__ = kernel
    return build


def _unary(kernel):
    def build(a):
        return make(kernel, [a])
    build.__name__ = kernel
    return build


add, sub, mul, div = _binary("add"), _binary("sub"), _binary("mul"), _binary("div")
pow = _binary("pow")  # noqa: A001
maximum = _binary("maximum")
lt, gt, le, ge, eq, neq = (_binary(k) for k in ("lt", "gt", "le", "ge", "eq", "neq"))
neg, exp, log, log1p = _unary("neg"), _unary("exp"), _unary("log"), _unary("log1p")
sqr, sqrt, sigmoid, tanh, isnan = (_unary(k) for k in ("sqr", "sqrt", "sigmoid", "tanh", "isnan"))


def switch(condition, a, b) -> Variable:
    return make("switch", [condition, a, b])


def infer_types(op, input_types):
    return op.infer_types(list(input_types))


def grad_rule(op, inputs, output_grads):
    return op.grad(list(inputs), list(output_grads))


def rop_rule(op, inputs, input_perturbations):
    return op.rop(list(inputs), list(input_perturbations))


def infer_shape(op, node, input_shapes):
    return op.infer_shape(node, list(input_shapes))


def perform(op, inputs, output_buffers=None):
    """Evaluate one op on host arrays (reference ``ops/base.py:118-120``).

    The reference runs ``op.perform`` on the CPU; here the op is executed on
    the B200 through a one-node compiled function (``preset="none"``: the op
    as given, no rewrites), so the reference's per-op golden tests exercise
    the device kernels.  Extent-1 dimensions are declared broadcastable, as
    the reference's NumPy broadcasting treats them.  ``output_buffers``, when
    given, receive the results (the reference's ``out=`` convention)."""
    import numpy as np

    from .dtypes import dtype_of_value
    from .graph import TensorType, Variable, apply
    from .vm import compile as _compile
    arrs = [np.asarray(v) for v in inputs]
    ins = [Variable(TensorType(dtype_of_value(a), tuple(d == 1 for d in a.shape))) for a in arrs]
    outs = apply(op, ins)
    res = _compile(ins, outs, preset="none")(*arrs)
    if output_buffers:
        for buf, r in zip(output_buffers, res):
            if buf is not None:
                np.copyto(buf, r)
        res = [buf if buf is not None else r for buf, r in zip(output_buffers, res)]
    return res


def conv2d_reference(x, f, stride=(1, 1), pad=(0, 0)):
    """Host-array cross-correlation with the reference algorithm's exact
    fp arithmetic (reference ``ops/conv.py:49-66``), computed on the device
    by the direct ``reference``-algorithm kernel."""
    from .conv import REFERENCE, Conv2d, FORWARD
    return perform(Conv2d(FORWARD, REFERENCE, tuple(stride), tuple(pad)), [x, f])[0]
