"""Elementwise operations and the fused Composite.

The 23 scalar kernels, their dtype rules, gradient and R-operator rules
follow reference ``ops/elemwise.py:84-157`` and ``:242-270``.  Execution is
different by design: every Elemwise / Composite node is lowered to a CUDA
kernel generated from hand-written templates (``codegen.py``) and compiled by
NVRTC for sm_100a; the scalar semantics each kernel must reproduce (NumPy's,
which the reference calls) are spelled out in ``codegen.KERNEL_CUDA``.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .dtypes import BOOL, is_float, np_dtype, promote_all
from .errors import TypeMismatch
from .graph import Constant, TensorType, Variable, apply, as_variable
from .op import (DISCONNECTED, UNKNOWN_SHAPE, Op, broadcast_pattern,
                 broadcast_shapes_checked, register_op)


@dataclass(frozen=True)
class ScalarKernel:
    name: str
    arity: int
    bool_out: bool = False


KERNELS = {k.name: k for k in [
    ScalarKernel("add", 2), ScalarKernel("sub", 2), ScalarKernel("mul", 2),
    ScalarKernel("div", 2), ScalarKernel("neg", 1), ScalarKernel("exp", 1),
    ScalarKernel("log", 1), ScalarKernel("log1p", 1), ScalarKernel("pow", 2),
    ScalarKernel("sqr", 1), ScalarKernel("sqrt", 1), ScalarKernel("sigmoid", 1),
    ScalarKernel("tanh", 1), ScalarKernel("maximum", 2), ScalarKernel("switch", 3),
    ScalarKernel("second", 2),
    ScalarKernel("lt", 2, True), ScalarKernel("gt", 2, True), ScalarKernel("le", 2, True),
    ScalarKernel("ge", 2, True), ScalarKernel("eq", 2, True), ScalarKernel("neq", 2, True),
    ScalarKernel("isnan", 1, True),
]}


def kernel_out_dtype(kernel: str, in_dtypes) -> str:
    if KERNELS[kernel].bool_out:
        return BOOL
    if kernel == "switch":
        return promote_all(in_dtypes[1:])
    return promote_all(in_dtypes)


def kernel_compute_dtype(kernel: str, in_dtypes) -> str:
    """dtype the operands are converted to before the scalar op runs."""
    if kernel == "switch":
        return promote_all(in_dtypes[1:])
    if kernel == "isnan":
        return in_dtypes[0]
    return promote_all(in_dtypes)


# -- compile-time folding of tiny constants (NumPy on host; never used to
#    execute a compiled function) ------------------------------------------

def _np_sigmoid(x):
    z = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + z), z / (1.0 + z))


def _np_div(a, b):
    if np.issubdtype(np.result_type(a, b), np.integer):
        if np.any(b == 0):
            raise ZeroDivisionError("integer division by zero")
        return np.floor_divide(a, b)
    return np.true_divide(a, b)


_FOLD = {
    "add": np.add, "sub": np.subtract, "mul": np.multiply, "div": _np_div,
    "neg": np.negative, "exp": np.exp, "log": np.log, "log1p": np.log1p,
    "pow": np.power, "sqr": np.square, "sqrt": np.sqrt, "sigmoid": _np_sigmoid,
    "tanh": np.tanh, "maximum": np.maximum, "switch": lambda c, a, b: np.where(c, a, b),
    "second": lambda a, b: np.broadcast_to(b, np.broadcast_shapes(a.shape, b.shape)).copy(),
    "lt": np.less, "gt": np.greater, "le": np.less_equal, "ge": np.greater_equal,
    "eq": np.equal, "neq": np.not_equal, "isnan": np.isnan,
}
FOLD_LIMIT = 4096  # elements


def fold_kernel(kernel, values, out_dtype):
    if any(np.asarray(v).size > FOLD_LIMIT for v in values):
        return None
    with np.errstate(all="ignore"):
        r = _FOLD[kernel](*values)
    return np.asarray(r).astype(np_dtype(out_dtype))


# -- gradient / R-op rules ----------------------------------------------

def _c(value, like: Variable) -> Constant:
    return Constant(value, dtype=like.type.dtype)


def _grad_pow(ins, v):
    x, y = ins
    return [v * y * make("pow", [x, y - _c(1, y)]),
            v * make("pow", [x, y]) * make("log", [x])]


def _grad_sigmoid(ins, v):
    s = make("sigmoid", ins)
    return [v * s * (_c(1, s) - s)]


def _grad_tanh(ins, v):
    t = make("tanh", ins)
    return [v * (_c(1, t) - make("sqr", [t]))]


GRADS = {
    "add": lambda ins, v: [v, v],
    "sub": lambda ins, v: [v, make("neg", [v])],
    "mul": lambda ins, v: [v * ins[1], v * ins[0]],
    "div": lambda ins, v: [v / ins[1], make("neg", [v * ins[0] / (ins[1] * ins[1])])],
    "neg": lambda ins, v: [make("neg", [v])],
    "exp": lambda ins, v: [v * make("exp", ins)],
    "log": lambda ins, v: [v / ins[0]],
    "log1p": lambda ins, v: [v / (ins[0] + _c(1, ins[0]))],
    "pow": _grad_pow,
    "sqr": lambda ins, v: [v * ins[0] * _c(2, ins[0])],
    "sqrt": lambda ins, v: [v / (make("sqrt", ins) * _c(2, ins[0]))],
    "sigmoid": _grad_sigmoid,
    "tanh": _grad_tanh,
    "maximum": lambda ins, v: [v * make("ge", ins), v * make("lt", ins)],
    "switch": lambda ins, v: [DISCONNECTED, make("switch", [ins[0], v, _c(0, v)]),
                              make("switch", [ins[0], _c(0, v), v])],
    "second": lambda ins, v: [DISCONNECTED, v],
}


def _sum_terms(terms):
    terms = [t for t in terms if t is not None]
    if not terms:
        return None
    return terms[0] if len(terms) == 1 else terms[0] + terms[1]


def _rop_unary(factor):
    return lambda ins, dx: [None if dx[0] is None else factor(ins[0]) * dx[0]]


def _rop_addsub(sign):
    def rule(ins, dx):
        a, b = dx
        if a is None and b is None:
            return [None]
        if a is None:
            return [make("neg", [b]) if sign < 0 else b]
        if b is None:
            return [a]
        return [a - b if sign < 0 else a + b]
    return rule


ROPS = {
    "add": _rop_addsub(1),
    "sub": _rop_addsub(-1),
    "mul": lambda ins, dx: [_sum_terms([None if dx[0] is None else dx[0] * ins[1],
                                        None if dx[1] is None else ins[0] * dx[1]])],
    "div": lambda ins, dx: [_sum_terms([
        None if dx[0] is None else dx[0] / ins[1],
        None if dx[1] is None else make("neg", [ins[0] * dx[1] / (ins[1] * ins[1])])])],
    "neg": lambda ins, dx: [None if dx[0] is None else make("neg", [dx[0]])],
    "exp": _rop_unary(lambda x: make("exp", [x])),
    "log": _rop_unary(lambda x: _c(1, x) / x),
    "log1p": _rop_unary(lambda x: _c(1, x) / (x + _c(1, x))),
    "pow": lambda ins, dx: [_sum_terms([
        None if dx[0] is None else ins[1] * make("pow", [ins[0], ins[1] - _c(1, ins[1])]) * dx[0],
        None if dx[1] is None else make("pow", ins) * make("log", [ins[0]]) * dx[1]])],
    "sqr": _rop_unary(lambda x: x * _c(2, x)),
    "sqrt": _rop_unary(lambda x: _c(1, x) / (make("sqrt", [x]) * _c(2, x))),
    "sigmoid": _rop_unary(lambda x: (lambda s: s * (_c(1, s) - s))(make("sigmoid", [x]))),
    "tanh": _rop_unary(lambda x: (lambda t: _c(1, t) - make("sqr", [t]))(make("tanh", [x]))),
    "maximum": lambda ins, dx: [None] if dx[0] is None and dx[1] is None else [make(
        "switch", [make("ge", ins), dx[0] if dx[0] is not None else _c(0, ins[0]),
                   dx[1] if dx[1] is not None else _c(0, ins[1])])],
    "switch": lambda ins, dx: [None] if dx[1] is None and dx[2] is None else [make(
        "switch", [ins[0], dx[1] if dx[1] is not None else _c(0, ins[1]),
                   dx[2] if dx[2] is not None else _c(0, ins[2])])],
    "second": lambda ins, dx: [None if dx[1] is None else make("second", [ins[0], dx[1]])],
}
for _k in ("lt", "gt", "le", "ge", "eq", "neq", "isnan"):
    ROPS[_k] = lambda ins, dx: [None]


# -- ops ------------------------------------------------------------------

def _broadcast_infer_shape(ndim, input_shapes):
    out = []
    for i in range(ndim):
        ext = None
        for s in input_shapes:
            if s is UNKNOWN_SHAPE:
                continue
            j = i - (ndim - len(s))
            if j < 0 or s[j] is None:
                continue
            if s[j] != 1:
                ext = s[j]
            elif ext is None:
                ext = 1
        out.append(ext)
    return tuple(out)


@register_op
class Elemwise(Op):
    """One scalar kernel lifted over tensors with right-aligned broadcasting."""

    name = "elemwise"
    inplace_capable = True
    fusable = True

    def __init__(self, kernel: str, destroy: int | None = None):
        if kernel not in KERNELS:
            raise TypeMismatch(f"unknown scalar kernel {kernel!r}")
        self.kernel = kernel
        self.destroy = destroy
        self.destroy_map = {} if destroy is None else {0: destroy}

    @property
    def display_name(self):
        return self.kernel + ("[inplace]" if self.destroy is not None else "")

    def attrs_key(self):
        return (self.kernel, self.destroy)

    def infer_types(self, input_types):
        spec = KERNELS[self.kernel]
        if len(input_types) != spec.arity:
            raise TypeMismatch(f"{self.kernel} expects {spec.arity} inputs, got {len(input_types)}")
        dt = kernel_out_dtype(self.kernel, [t.dtype for t in input_types])
        return [TensorType(dt, broadcast_pattern([t.broadcastable for t in input_types]))]

    def check_runtime_shapes(self, node, shapes):
        broadcast_shapes_checked(node, shapes)

    def infer_shape(self, node, input_shapes):
        return [_broadcast_infer_shape(node.outputs[0].type.ndim, input_shapes)]

    def grad(self, inputs, output_grads):
        (v,) = output_grads
        out_dt = self.infer_types([x.type for x in inputs])[0].dtype
        if self.kernel not in GRADS or not is_float(out_dt):
            return [DISCONNECTED] * len(inputs)
        raw = GRADS[self.kernel](inputs, v)
        return [DISCONNECTED if g is DISCONNECTED or not is_float(x.type.dtype)
                else sum_to_matching_shape(g, x) for x, g in zip(inputs, raw)]

    def rop(self, inputs, input_perturbations):
        return ROPS[self.kernel](inputs, input_perturbations)

    def fold(self, values):
        r = fold_kernel(self.kernel, values, kernel_out_dtype(self.kernel, [str(v.dtype) for v in values]))
        return None if r is None else [r]

    def lower(self, node, plan):
        from . import codegen
        codegen.lower_elementwise(node, plan, EwProgram.single(self.kernel, [x.type.dtype for x in node.inputs]))

    def attrs_payload(self, encode_graph=None):
        d = {"kernel": self.kernel}
        if self.destroy is not None:
            d["destroy"] = self.destroy
        return d

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["kernel"], payload.get("destroy"))


def make(kernel: str, args: Sequence) -> Variable:
    """Apply a scalar kernel; Python numbers take the dtype of the first
    variable argument when that is lossless (reference ``ops/elemwise.py:374-395``)."""
    anchor = next((a for a in args if isinstance(a, Variable)), None)
    vs = []
    for a in args:
        if isinstance(a, Variable):
            vs.append(a)
        elif anchor is not None and isinstance(a, (bool, int)) and not isinstance(a, np.ndarray):
            vs.append(Constant(a, dtype=anchor.type.dtype))
        elif anchor is not None and isinstance(a, float) and is_float(anchor.type.dtype):
            vs.append(Constant(a, dtype=anchor.type.dtype))
        else:
            vs.append(as_variable(a))
    return apply(Elemwise(kernel), vs)[0]


def fill(template: Variable, value) -> Variable:
    return make("second", [template, value])


def zeros_like(x: Variable) -> Variable:
    return fill(x, _c(0, x))


def ones_like(x: Variable) -> Variable:
    return fill(x, _c(1, x))


def sum_to_matching_shape(g: Variable, target: Variable) -> Variable:
    """Undo broadcasting in a gradient: sum the leading dims ``target`` lacks
    and the dims where ``target`` is guaranteed-1 but ``g`` is not, then
    re-insert unit axes (reference ``ops/elemwise.py:411-442``)."""
    from . import reduce as _reduce
    from .shaping import dimshuffle

    tp, gp = target.type.broadcastable, g.type.broadcastable
    lead = len(gp) - len(tp)
    axes = list(range(lead))
    unit = [i for i, b in enumerate(tp) if b and not gp[lead + i]]
    axes += [lead + i for i in unit]
    if not axes:
        return g
    r = _reduce.sum(g, axis=tuple(axes))
    if not unit:
        return r
    pattern, k = [], 0
    for i in range(len(tp)):
        if i in unit:
            pattern.append("x")
        else:
            pattern.append(k)
            k += 1
    return dimshuffle(r, tuple(pattern))


# -- the fused program ------------------------------------------------------

class EwProgram:
    """A scalar DAG in canonical, hashable form: the NVRTC cache key.

    ``in_dtypes``: leaf dtypes; ``consts``: tuple of (dtype, python value);
    ``nodes``: tuple of (kernel, refs, out_dtype) with refs ("in", i) /
    ("const", j) / ("node", j); ``outputs``: tuple of refs.  Mirrors the
    reference Composite payload (``ops/elemwise.py:646-673``).
    """

    __slots__ = ("in_dtypes", "consts", "nodes", "outputs", "_key")

    def __init__(self, in_dtypes, consts, nodes, outputs):
        self.in_dtypes = tuple(in_dtypes)
        self.consts = tuple(consts)
        self.nodes = tuple((k, tuple(map(tuple, refs)), dt) for k, refs, dt in nodes)
        self.outputs = tuple(tuple(r) for r in outputs)
        self._key = (self.in_dtypes, self.consts, self.nodes, self.outputs)

    @classmethod
    def single(cls, kernel, in_dtypes):
        return cls(in_dtypes, (), [(kernel, [("in", i) for i in range(len(in_dtypes))],
                                    kernel_out_dtype(kernel, list(in_dtypes)))], [("node", 0)])

    def ref_dtype(self, ref):
        kind, i = ref
        if kind == "in":
            return self.in_dtypes[i]
        if kind == "const":
            return self.consts[i][0]
        return self.nodes[i][2]

    @property
    def out_dtypes(self):
        return tuple(self.ref_dtype(r) for r in self.outputs)

    def key(self):
        return self._key

    def __eq__(self, o):
        return isinstance(o, EwProgram) and o._key == self._key

    def __hash__(self):
        return hash(self._key)

    def __len__(self):
        return len(self.nodes)


@register_op
class CompositeElemwise(Op):
    """One node evaluating a fused scalar DAG per element (reference
    ``CompositeElemwise``, ``ops/elemwise.py:452-695``).  Built by the convex
    fusion pass; lowered to one generated kernel."""

    name = "composite"
    fusable = True

    def __init__(self, program: EwProgram):
        self.program = program

    @property
    def display_name(self):
        return f"composite[{len(self.program)}]"

    def attrs_key(self):
        return (self.program.key(),)

    def _leaves_of_outputs(self):
        p = self.program
        res = []
        for r in p.outputs:
            seen, stack, leaves = set(), [r], set()
            while stack:
                kind, i = stack.pop()
                if (kind, i) in seen:
                    continue
                seen.add((kind, i))
                if kind == "in":
                    leaves.add(i)
                elif kind == "node":
                    stack.extend(p.nodes[i][1])
            res.append(sorted(leaves))
        return res

    def infer_types(self, input_types):
        p = self.program
        if len(input_types) != len(p.in_dtypes):
            raise TypeMismatch("composite arity mismatch")
        for t, d in zip(input_types, p.in_dtypes):
            if t.dtype != d:
                raise TypeMismatch(f"composite input dtype {t.dtype} != expected {d}")
        out = []
        for dt, leaves in zip(p.out_dtypes, self._leaves_of_outputs()):
            out.append(TensorType(dt, broadcast_pattern([input_types[i].broadcastable for i in leaves])
                                  if leaves else ()))
        return out

    def check_runtime_shapes(self, node, shapes):
        broadcast_shapes_checked(node, shapes)

    def infer_shape(self, node, input_shapes):
        leaves = self._leaves_of_outputs()
        return [_broadcast_infer_shape(o.type.ndim, [input_shapes[i] for i in lv])
                for o, lv in zip(node.outputs, leaves)]

    def rebuild(self, inputs):
        """Re-express as plain Elemwise nodes (used by grad / rop)."""
        p = self.program
        vals = []
        consts = [Constant(v, dtype=d) for d, v in p.consts]

        def get(ref):
            kind, i = ref
            return inputs[i] if kind == "in" else consts[i] if kind == "const" else vals[i]

        for k, refs, _ in p.nodes:
            vals.append(apply(Elemwise(k), [get(r) for r in refs])[0])
        return [get(r) for r in p.outputs]

    def grad(self, inputs, output_grads):
        from . import autodiff
        return autodiff.lop(self.rebuild(inputs), output_grads, inputs)

    def rop(self, inputs, input_perturbations):
        from . import autodiff
        return autodiff.forward_perturbations(self.rebuild(inputs), dict(zip(inputs, input_perturbations)))

    def lower(self, node, plan):
        from . import codegen
        codegen.lower_elementwise(node, plan, self.program)

    def attrs_payload(self, encode_graph=None):
        p = self.program
        return {"inputs": [{"dtype": d} for d in p.in_dtypes],
                "consts": [{"dtype": d, "value": v} for d, v in p.consts],
                "nodes": [{"kernel": k, "inputs": [list(r) for r in refs]} for k, refs, _ in p.nodes],
                "outputs": [list(r) for r in p.outputs]}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        in_dt = [e["dtype"] for e in payload["inputs"]]
        consts = [(e["dtype"], e["value"]) for e in payload["consts"]]
        nodes = []
        tmp = EwProgram(in_dt, consts, [], [])
        for e in payload["nodes"]:
            refs = [tuple(r) for r in e["inputs"]]
            dts = [tmp.ref_dtype(r) if r[0] != "node" else nodes[r[1]][2] for r in refs]
            nodes.append((e["kernel"], refs, kernel_out_dtype(e["kernel"], dts)))
        return cls(EwProgram(in_dt, consts, nodes, [tuple(r) for r in payload["outputs"]]))


# Reference name, kept for drop-in imports.
Composite = CompositeElemwise
