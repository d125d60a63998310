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
