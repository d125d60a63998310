"""Axis shuffles as zero-copy device views.

``DimShuffle`` follows reference ``ops/shaping.py:17-94`` (pattern of input
dims and ``'x'`` fresh unit axes; unreferenced dims must be guaranteed
extent 1).  On the device it never launches a kernel: the output is the
input's buffer with permuted strides (stride 0 on inserted axes), so a
transposed operand reaches the GEMM as a layout flag, not a copy.
"""
from __future__ import annotations

import numpy as np

from .dtypes import is_float
from .errors import TypeMismatch
from .graph import TensorType, Variable, apply
from .op import DISCONNECTED, UNKNOWN_SHAPE, Op, register_op


@register_op
class DimShuffle(Op):
    name = "dimshuffle"
    view_capable = True
    view_map = {0: 0}

    def __init__(self, pattern):
        self.pattern = tuple(pattern)
        for p in self.pattern:
            if p != "x" and not isinstance(p, (int, np.integer)):
                raise TypeMismatch(f"bad dimshuffle pattern entry {p!r}")
        self.pattern = tuple(p if p == "x" else int(p) for p in self.pattern)

    @property
    def display_name(self):
        return f"dimshuffle{self.pattern}"

    def attrs_key(self):
        return (self.pattern,)

    def kept(self):
        return [p for p in self.pattern if p != "x"]

    def infer_types(self, input_types):
        (t,) = input_types
        kept = self.kept()
        if len(set(kept)) != len(kept):
            raise TypeMismatch("dimshuffle pattern repeats a dimension")
        for d in kept:
            if not 0 <= d < t.ndim:
                raise TypeMismatch(f"dimshuffle dim {d} out of range for rank {t.ndim}")
        for i in range(t.ndim):
            if i not in kept and not t.broadcastable[i]:
                raise TypeMismatch(f"dimshuffle drops dim {i} which is not guaranteed extent 1")
        return [TensorType(t.dtype, tuple(True if p == "x" else t.broadcastable[p]
                                          for p in self.pattern))]

    def infer_shape(self, node, input_shapes):
        (s,) = input_shapes
        if s is UNKNOWN_SHAPE:
            return [UNKNOWN_SHAPE]
        return [tuple(1 if p == "x" else s[p] for p in self.pattern)]

    def view_layout(self, node, in_layouts):
        (shape, strides, offset) = in_layouts[0]
        return (tuple(1 if p == "x" else shape[p] for p in self.pattern),
                tuple(0 if p == "x" else strides[p] for p in self.pattern), offset)

    def grad(self, inputs, output_grads):
        (x,), (v,) = inputs, output_grads
        if not is_float(x.type.dtype):
            return [DISCONNECTED]
        inv = tuple(self.pattern.index(i) if i in self.pattern else "x" for i in range(x.type.ndim))
        return [dimshuffle(v, inv)]

    def rop(self, inputs, input_perturbations):
        (dx,) = input_perturbations
        return [None if dx is None else dimshuffle(dx, self.pattern)]

    def fold(self, values):
        (x,) = values
        kept = self.kept()
        dropped = [i for i in range(x.ndim) if i not in kept]
        y = np.transpose(x, kept + dropped)
        idx = tuple([None if p == "x" else slice(None) for p in self.pattern] + [0] * len(dropped))
        return [np.ascontiguousarray(y[idx])]

    def attrs_payload(self, encode_graph=None):
        return {"pattern": list(self.pattern)}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(tuple(p if p == "x" else int(p) for p in payload["pattern"]))


def dimshuffle(x: Variable, pattern) -> Variable:
    return apply(DimShuffle(pattern), [x])[0]


def transpose(x: Variable, axes=None) -> Variable:
    if axes is None:
        axes = tuple(reversed(range(x.type.ndim)))
    return dimshuffle(x, tuple(axes))
