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
        return [np.asarray(y[idx], order="C")]

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


# ---------------------------------------------------------------------------
# Basic slicing, increment-into-slice and concatenation (reference
# ``ops/shaping.py:107-479``).  On the device a slice is a view (offset plus
# strides, negative for reversed steps), ``inc_subtensor`` is a copy followed
# by an in-place add over the sliced view, and ``join`` copies each piece into
# its slab of the output.  They exist for symbolic loops (``scan.py``): the
# reversed-sequence streams of backpropagation through time.

def _norm_item(item, what="index"):
    if isinstance(item, (bool, np.bool_)):
        raise TypeMismatch(f"unsupported {what} entry {item!r} (basic slicing only)")
    if isinstance(item, (int, np.integer)):
        return int(item)
    if isinstance(item, (tuple, list)) and len(item) == 3:
        return tuple(None if v is None else int(v) for v in item)
    if isinstance(item, slice):
        return tuple(None if v is None else int(v) for v in (item.start, item.stop, item.step))
    raise TypeMismatch(f"unsupported {what} entry {item!r} (basic slicing only)")


def _is_full_slice(entry):
    return entry in ((None, None, None), (None, None, 1))


def _slice_geometry(items, shape, strides, offset):
    """(shape, strides, offset) of x[items] for a strided layout; raises
    ShapeMismatch on an out-of-range integer index (NumPy's IndexError)."""
    from .errors import ShapeMismatch
    out_shape, out_strides = [], []
    for i, item in enumerate(items):
        n, st = shape[i], strides[i]
        if isinstance(item, int):
            j = item + n if item < 0 else item
            if not 0 <= j < n:
                raise ShapeMismatch(f"subtensor index {item} out of bounds for axis {i} with size {n}")
            offset += j * st
            continue
        start, stop, step = slice(*item).indices(n)
        length = len(range(start, stop, step))
        if length > 0:
            offset += start * st
        out_shape.append(length)
        out_strides.append(st * step)
    out_shape.extend(shape[len(items):])
    out_strides.extend(strides[len(items):])
    return tuple(out_shape), tuple(out_strides), offset


@register_op
class Subtensor(Op):
    """Basic slicing: per dim an integer index or a (start, stop, step)
    triple (None = unspecified).  A zero-copy view on the device."""

    name = "subtensor"
    view_capable = True
    view_map = {0: 0}

    def __init__(self, items):
        self.items = tuple(_norm_item(i) for i in items)

    @property
    def display_name(self):
        return f"subtensor{self.items}"

    def attrs_key(self):
        return (self.items,)

    def infer_types(self, input_types):
        (t,) = input_types
        if len(self.items) > t.ndim:
            raise TypeMismatch(f"{len(self.items)} index entries for rank {t.ndim}")
        out = []
        for i, item in enumerate(self.items):
            if isinstance(item, int):
                continue
            out.append(t.broadcastable[i] if _is_full_slice(item) else False)
        out.extend(t.broadcastable[len(self.items):])
        return [TensorType(t.dtype, tuple(out))]

    def infer_shape(self, node, input_shapes):
        (s,) = input_shapes
        if s is UNKNOWN_SHAPE:
            return [UNKNOWN_SHAPE]
        out = []
        for i, item in enumerate(self.items):
            if isinstance(item, int):
                continue
            out.append(None if s[i] is None else len(range(*slice(*item).indices(s[i]))))
        out.extend(s[len(self.items):])
        return [tuple(out)]

    def check_runtime_shapes(self, node, shapes):
        _slice_geometry(self.items, shapes[0], (0,) * len(shapes[0]), 0)

    def view_layout(self, node, in_layouts):
        shape, strides, offset = in_layouts[0]
        return _slice_geometry(self.items, shape, strides, offset)

    def grad(self, inputs, output_grads):
        from .elemwise import zeros_like
        (x,), (v,) = inputs, output_grads
        if not is_float(x.type.dtype):
            return [DISCONNECTED]
        return [inc_subtensor(zeros_like(x), v, self.items)]

    def rop(self, inputs, input_perturbations):
        (dx,) = input_perturbations
        return [None if dx is None else apply(Subtensor(self.items), [dx])[0]]

    def fold(self, values):
        (x,) = values
        return [np.asarray(x[tuple(i if isinstance(i, int) else slice(*i) for i in self.items)], order="C")]

    def attrs_payload(self, encode_graph=None):
        return {"items": [i if isinstance(i, int) else list(i) for i in self.items]}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(tuple(i if isinstance(i, int) else tuple(i) for i in payload["items"]))


def subtensor(x: Variable, key) -> Variable:
    if not isinstance(key, tuple):
        key = (key,)
    return apply(Subtensor(key), [x])[0]


def flip0(x: Variable) -> Variable:
    """Reverse along the leading axis (a negative-stride view)."""
    return subtensor(x, (slice(None, None, -1),))


@register_op
class IncSubtensor(Op):
    """Copy of ``target`` with ``value`` added into the indexed region
    (NumPy ``out[idx] += value``, value broadcast to the region)."""

    name = "inc_subtensor"

    def __init__(self, items):
        self.items = tuple(_norm_item(i) for i in items)

    @property
    def display_name(self):
        return f"inc_subtensor{self.items}"

    def attrs_key(self):
        return (self.items,)

    def infer_types(self, input_types):
        target, value = input_types
        probe = Subtensor(self.items).infer_types([target])[0]
        if probe.dtype != value.dtype or probe.ndim != value.ndim:
            raise TypeMismatch(f"inc_subtensor value {value} does not match region type {probe}")
        return [target]

    def infer_shape(self, node, input_shapes):
        return [input_shapes[0]]

    def check_runtime_shapes(self, node, shapes):
        from .errors import ShapeMismatch
        region, _, _ = _slice_geometry(self.items, shapes[0], (0,) * len(shapes[0]), 0)
        v = shapes[1]
        for r, e in zip(reversed(region), reversed(v)):
            if e != r and e != 1:
                raise ShapeMismatch(f"inc_subtensor value of shape {tuple(v)} does not broadcast to region {region}")

    def grad(self, inputs, output_grads):
        (v,) = output_grads
        out = []
        for i, x in enumerate(inputs):
            if not is_float(x.type.dtype):
                out.append(DISCONNECTED)
            elif i == 0:
                out.append(v)
            else:
                out.append(apply(Subtensor(self.items), [v])[0])
        return out

    def rop(self, inputs, input_perturbations):
        from .elemwise import zeros_like
        dt, dv = input_perturbations
        if dt is None and dv is None:
            return [None]
        dt = dt if dt is not None else zeros_like(inputs[0])
        return [dt if dv is None else inc_subtensor(dt, dv, self.items)]

    def lower(self, node, plan):
        from .elemwise import EwProgram
        out, target, value = node.outputs[0], node.inputs[0], node.inputs[1]
        lo, lt, lv = plan.layout(out), plan.layout(target), plan.layout(value)
        if lo.storage.root() is not lt.storage.root() or lo.offset != lt.offset or lo.strides != lt.strides:
            plan.emit_copy_layouts(lt, lo)
        shape, strides, off = _slice_geometry(self.items, lo.shape, lo.strides, lo.offset)
        if 0 in shape:
            return
        region = plan.view_of(lo, shape, strides, off)
        vs = [0] * len(shape)
        for k in range(1, len(lv.shape) + 1):
            vs[-k] = 0 if lv.shape[-k] == 1 else lv.strides[-k]
        dt = out.type.dtype
        prog = EwProgram.single("add", [dt, dt])
        plan.emit_elementwise_tx(prog, [plan.tx(region)], [plan.tx(region), plan.tx(lv, shape, tuple(vs))])

    def attrs_payload(self, encode_graph=None):
        return {"items": [i if isinstance(i, int) else list(i) for i in self.items]}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(tuple(i if isinstance(i, int) else tuple(i) for i in payload["items"]))


def _as_index(items):
    return tuple(i if isinstance(i, int) else slice(*i) for i in items)


@register_op
class ZeroEmbed(Op):
    """zeros of ``template``'s shape with each value added into its region:
    ``inc_subtensor(...inc_subtensor(zeros_like(template), v0, r0)..., vk, rk)``
    as one node (B200-specific; built by ``scan.loop_body_zero_embed`` from
    the region-embedded gradient sums ``grad`` writes, e.g. the LSTM's four
    gate gradients).  When the regions partition the output at plan time,
    each value's producer writes straight into its region (``StepPlan``
    places it) and the node costs nothing; otherwise it zero-fills and adds.
    ``expand`` gives the reference-op chain for portable saves."""

    name = "zero_embed"

    def __init__(self, regions):
        self.regions = tuple(tuple(_norm_item(i) for i in items) for items in regions)

    @property
    def display_name(self):
        return f"zero_embed[{len(self.regions)}]"

    def attrs_key(self):
        return (self.regions,)

    def infer_types(self, input_types):
        target = input_types[0]
        for items, value in zip(self.regions, input_types[1:]):
            IncSubtensor(items).infer_types([target, value])
        return [target]

    def infer_shape(self, node, input_shapes):
        return [input_shapes[0]]

    def check_runtime_shapes(self, node, shapes):
        for items, v in zip(self.regions, shapes[1:]):
            IncSubtensor(items).check_runtime_shapes(node, [shapes[0], v])

    def partition(self, shape):
        """Whether the regions (at this concrete shape) are disjoint, cover the
        whole tensor, and each value fills its region exactly."""
        cover = np.zeros(shape, dtype=np.int32) if int(np.prod(shape, dtype=np.int64)) <= (1 << 22) else None
        if cover is None:
            return False
        for items in self.regions:
            cover[_as_index(items)] += 1
        return bool(np.all(cover == 1))

    def grad(self, inputs, output_grads):
        (v,) = output_grads
        out = [DISCONNECTED]
        for items, x in zip(self.regions, inputs[1:]):
            out.append(apply(Subtensor(items), [v])[0] if is_float(x.type.dtype) else DISCONNECTED)
        return out

    def rop(self, inputs, input_perturbations):
        from .elemwise import zeros_like
        dvs = input_perturbations[1:]
        if all(d is None for d in dvs):
            return [None]
        acc = zeros_like(inputs[0])
        for items, d in zip(self.regions, dvs):
            if d is not None:
                acc = inc_subtensor(acc, d, items)
        return [acc]

    def expand(self, inputs):
        """The reference-op form: zeros_like(template) and a chain of inc_subtensors."""
        from .elemwise import zeros_like
        acc = zeros_like(inputs[0])
        for items, v in zip(self.regions, inputs[1:]):
            acc = inc_subtensor(acc, v, items)
        return [acc]

    def fold(self, values):
        out = np.zeros(np.shape(values[0]), dtype=np.asarray(values[0]).dtype)
        for items, v in zip(self.regions, values[1:]):
            out[_as_index(items)] += v
        return [out]

    def lower(self, node, plan):
        from .elemwise import EwProgram
        out = node.outputs[0]
        lo = plan.layout(out)
        placed = plan.placed.get(node.id, ()) if hasattr(plan, "placed") else ()
        part = self.partition(lo.shape)
        if not part:
            plan.emit_fill_zero(lo)
        dt = out.type.dtype
        for k, (items, v) in enumerate(zip(self.regions, node.inputs[1:])):
            if k in placed:
                continue  # its producer wrote the region already
            lv = plan.layout(v)
            shape, strides, off = _slice_geometry(items, lo.shape, lo.strides, lo.offset)
            if 0 in shape:
                continue
            region = plan.view_of(lo, shape, strides, off)
            vs = [0] * len(shape)
            for j in range(1, len(lv.shape) + 1):
                vs[-j] = 0 if lv.shape[-j] == 1 else lv.strides[-j]
            if part:
                plan.emit_copy_layouts(plan.view_of(lv, shape, tuple(vs), lv.offset), region)
            else:
                plan.emit_elementwise_tx(EwProgram.single("add", [dt, dt]), [plan.tx(region)],
                                         [plan.tx(region), plan.tx(lv, shape, tuple(vs))])

    def attrs_payload(self, encode_graph=None):
        return {"regions": [[i if isinstance(i, int) else list(i) for i in items] for items in self.regions]}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(tuple(tuple(i if isinstance(i, int) else tuple(i) for i in items) for items in payload["regions"]))


def inc_subtensor(target: Variable, value: Variable, items) -> Variable:
    return apply(IncSubtensor(items), [target, value])[0]


@register_op
class Join(Op):
    """Concatenate along one axis (reference ``ops/shaping.py:381-470``);
    differentiable when every piece is guaranteed extent 1 on the axis."""

    name = "join"

    def __init__(self, axis: int):
        self.axis = int(axis)

    @property
    def display_name(self):
        return f"join[{self.axis}]"

    def attrs_key(self):
        return (self.axis,)

    def infer_types(self, input_types):
        if not input_types:
            raise TypeMismatch("join of nothing")
        ndim, dtype = input_types[0].ndim, input_types[0].dtype
        for t in input_types:
            if t.ndim != ndim or t.dtype != dtype:
                raise TypeMismatch("join inputs must share rank and dtype")
        if not 0 <= self.axis < ndim:
            raise TypeMismatch(f"join axis {self.axis} out of range for rank {ndim}")
        return [TensorType(dtype, tuple(all(t.broadcastable[i] for t in input_types) and i != self.axis
                                        for i in range(ndim)))]

    def infer_shape(self, node, input_shapes):
        if any(s is UNKNOWN_SHAPE for s in input_shapes):
            return [UNKNOWN_SHAPE]
        out = []
        for i in range(node.outputs[0].type.ndim):
            dims = [s[i] for s in input_shapes]
            if i == self.axis:
                out.append(None if any(d is None for d in dims) else sum(dims))
            else:
                known = [d for d in dims if d is not None]
                out.append(known[0] if known else None)
        return [tuple(out)]

    def check_runtime_shapes(self, node, shapes):
        from .errors import ShapeMismatch
        for i in range(len(shapes[0])):
            if i != self.axis and len({s[i] for s in shapes}) > 1:
                raise ShapeMismatch(f"join: pieces disagree on axis {i}: {[s[i] for s in shapes]}")

    def grad(self, inputs, output_grads):
        from .elemwise import sum_to_matching_shape
        from .errors import NotDifferentiable
        (v,) = output_grads
        if any(not x.type.broadcastable[self.axis] for x in inputs):
            raise NotDifferentiable("join gradient needs guaranteed extent-1 pieces along the axis "
                                    "(general split boundaries are runtime values)")
        grads = []
        for i, x in enumerate(inputs):
            if not is_float(x.type.dtype):
                grads.append(DISCONNECTED)
                continue
            piece = apply(Subtensor(((None, None, None),) * self.axis + (i,)), [v])[0]
            pattern = list(range(piece.type.ndim))
            pattern.insert(self.axis, "x")
            grads.append(sum_to_matching_shape(dimshuffle(piece, tuple(pattern)), x))
        return grads

    def rop(self, inputs, input_perturbations):
        from .elemwise import zeros_like
        if all(p is None for p in input_perturbations):
            return [None]
        return [apply(Join(self.axis), [p if p is not None else zeros_like(x)
                                        for x, p in zip(inputs, input_perturbations)])[0]]

    def lower(self, node, plan):
        lo = plan.layout(node.outputs[0])
        at = 0
        for x in node.inputs:
            lx = plan.layout(x)
            n = lx.shape[self.axis]
            if n:
                shape = lo.shape[:self.axis] + (n,) + lo.shape[self.axis + 1:]
                dst = plan.view_of(lo, shape, lo.strides, lo.offset + at * lo.strides[self.axis])
                plan.emit_copy_layouts(lx, dst)
            at += n

    def fold(self, values):
        return [np.concatenate(values, axis=self.axis)]

    def attrs_payload(self, encode_graph=None):
        return {"axis": self.axis}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["axis"])


def join(axis: int, *tensors: Variable) -> Variable:
    return apply(Join(axis), list(tensors))[0]


# ---------------------------------------------------------------------------
# Runtime shape vectors and reshape (reference ``ops/shaping.py:281-378``).
# Step plans know every shape before launching, so a ``shape_of`` value is a
# plan-time constant (uploaded once per plan) and ops that take shape vectors
# (reshape, the convolution gradients) read it at planning time.

@register_op
class ShapeOf(Op):
    """Runtime shape of a tensor as an int64 vector of static length."""

    name = "shape_of"
    plan_value = True

    def infer_types(self, input_types):
        (t,) = input_types
        return [TensorType("int64", (t.ndim == 1,))]

    def infer_shape(self, node, input_shapes):
        return [(node.inputs[0].type.ndim,)]

    def value(self, node, input_shapes):
        return np.asarray(input_shapes[0], dtype=np.int64)

    def grad(self, inputs, output_grads):
        return [DISCONNECTED]

    def rop(self, inputs, input_perturbations):
        return [None]

    def lower(self, node, plan):
        from .graph import Constant
        c = Constant(plan.values[node.outputs[0].id], dtype="int64")
        plan.emit_copy_layouts(plan._const_layout(c), plan.layout(node.outputs[0]))


def shape_of(x: Variable) -> Variable:
    return apply(ShapeOf(), [x])[0]


def _shape_arg(node, k, values):
    from .graph import Constant
    v = node.inputs[k]
    if isinstance(v, Constant):
        return tuple(int(s) for s in v.value)
    if values is not None and v.id in values:
        return tuple(int(s) for s in values[v.id])
    return None


@register_op
class Reshape(Op):
    """Reshape against a shape vector; the output rank is static."""

    name = "reshape"
    uses_values = True

    def __init__(self, ndim: int):
        self.ndim = int(ndim)

    @property
    def display_name(self):
        return f"reshape{{{self.ndim}}}"

    def attrs_key(self):
        return (self.ndim,)

    def infer_types(self, input_types):
        x, shp = input_types
        if shp.ndim != 1 or shp.dtype not in ("int32", "int64"):
            raise TypeMismatch("reshape expects a 1-d integer shape vector")
        return [TensorType(x.dtype, (False,) * self.ndim)]

    def infer_shape(self, node, input_shapes, values=None):
        from .errors import ShapeMismatch
        dims = _shape_arg(node, 1, values)
        if dims is None:
            return [(None,) * self.ndim]
        xs = input_shapes[0]
        if xs is UNKNOWN_SHAPE or any(d is None for d in xs):
            return [dims if -1 not in dims else (None,) * self.ndim]
        total = int(np.prod(xs, dtype=np.int64))
        if dims.count(-1) == 1:
            known = int(np.prod([d for d in dims if d != -1], dtype=np.int64))
            if known == 0 or total % known:
                raise ShapeMismatch(f"reshape: cannot reshape {tuple(xs)} to {dims}")
            dims = tuple(total // known if d == -1 else d for d in dims)
        if len(dims) != self.ndim or int(np.prod(dims, dtype=np.int64)) != total:
            raise ShapeMismatch(f"reshape: cannot reshape {tuple(xs)} to {dims}")
        return [dims]

    def grad(self, inputs, output_grads):
        x, _ = inputs
        (v,) = output_grads
        if not is_float(x.type.dtype):
            return [DISCONNECTED, DISCONNECTED]
        return [reshape(v, shape_of(x), ndim=x.type.ndim), DISCONNECTED]

    def rop(self, inputs, input_perturbations):
        dx, _ = input_perturbations
        return [None if dx is None else reshape(dx, inputs[1], ndim=self.ndim)]

    def lower(self, node, plan):
        from .vm import contiguous_strides
        lx, lo = plan.layout(node.inputs[0]), plan.layout(node.outputs[0])
        if lo.numel == 0:
            return
        if not lx.contiguous():
            tmp = plan.scratch(lx.shape, lx.dtype)
            plan.emit_copy_layouts(lx, tmp)
            lx = tmp
        src = plan.view_of(lx, lo.shape, contiguous_strides(lo.shape), lx.offset)
        plan.emit_copy_layouts(src, lo)

    def attrs_payload(self, encode_graph=None):
        return {"ndim": self.ndim}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["ndim"])


def reshape(x: Variable, shape, ndim: int | None = None) -> Variable:
    from .graph import as_variable
    if isinstance(shape, (tuple, list)):
        ndim = len(shape)
        shape = as_variable(np.asarray(shape, dtype=np.int64))
    elif ndim is None:
        raise TypeMismatch("reshape with a symbolic shape needs an explicit ndim")
    return apply(Reshape(ndim), [x, shape])[0]
