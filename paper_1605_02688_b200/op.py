"""The operator plugin contract and broadcasting helpers.

Same surface as reference ``ops/base.py:37-111`` (``infer_types``,
``check_runtime_shapes``, ``grad``, ``rop``, ``infer_shape``, ``attrs_key``
value identity, ``attrs_payload``/``from_payload``, capability flags, and the
``register_op`` registry) with one substitution: built-in ops have no host
``perform``.  An op executes by *lowering* onto the device — ``lower(node, plan)`` appends
launches of hand-written sm_100a kernels to a step plan (see ``vm.py``), or the
op declares itself a zero-copy view (``view_layout``).  ``fold`` is a
compile-time constant-folding hook restricted to tiny constants; it is never
used to execute a compiled function.  A *user* op that only implements the
reference's host ``perform`` still runs, as a host step (``is_host_op``).
"""
from __future__ import annotations

from typing import Sequence

from .errors import NotDifferentiable, NotSupported, ShapeMismatch, TypeMismatch
from .graph import TensorType


class _Marker:
    def __init__(self, text):
        self._text = text

    def __repr__(self):
        return self._text


DISCONNECTED = _Marker("<disconnected>")
UNKNOWN_SHAPE = _Marker("<unknown-shape>")


class Op:
    name = "op"
    has_grad = True
    has_rop = True
    inplace_capable = False
    view_capable = False
    lazy = False
    fusable = False
    foldable = True
    destroy_map: dict = {}
    view_map: dict = {}

    # value identity ------------------------------------------------------
    def attrs_key(self) -> tuple:
        return ()

    def __eq__(self, other):
        return type(self) is type(other) and self.attrs_key() == other.attrs_key()

    def __hash__(self):
        return hash((type(self).__name__, self.attrs_key()))

    def __repr__(self):
        return f"<op {getattr(self, 'display_name', self.name)}>"

    # typing / shapes -----------------------------------------------------
    def infer_types(self, input_types: Sequence[TensorType]) -> list[TensorType]:
        raise NotImplementedError

    def check_runtime_shapes(self, node, shapes) -> None:
        """Raise ShapeMismatch when concrete input shapes are incompatible."""

    def infer_shape(self, node, input_shapes) -> list:
        return [UNKNOWN_SHAPE for _ in node.outputs]

    # differentiation -----------------------------------------------------
    def grad(self, inputs, output_grads) -> list:
        raise NotDifferentiable(f"op {self.name} has no gradient rule")

    def rop(self, inputs, input_perturbations) -> list:
        raise NotSupported(f"op {self.name} has no R-operator rule")

    # device execution ----------------------------------------------------
    def view_layout(self, node, in_layouts):
        """For view ops: output (shape, strides, offset) from the input's."""
        raise NotImplementedError

    def lower(self, node, plan) -> None:
        if is_host_op(self):
            plan.emit_host_op(node)
            return
        raise NotSupported(f"op {self.name} has no B200 lowering")

    def perform(self, inputs, output_buffers=None):
        """Host evaluation -- only for user plugin ops (see ``is_host_op``);
        every built-in op lowers to device kernels instead."""
        raise NotSupported(f"op {self.name} has no host perform (it executes on the device via lower)")

    def fold(self, values):
        """Compile-time evaluation on tiny host constants, or None."""
        return None

    # serialization -------------------------------------------------------
    def attrs_payload(self, encode_graph=None) -> dict:
        return {}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls()


def is_host_op(op) -> bool:
    """A user plugin op written against the reference's contract only
    (``perform`` on host arrays, reference ``ops/base.py:37-111``) and no
    device ``lower``.  The VM runs such a node as a host step inside the
    device step: the stream is drained, the node's inputs come to the host,
    ``perform`` runs, its outputs go back to the planned device buffers, and
    the step is not captured as a CUDA graph.  None of the built-in ops is a
    host op: the hot path is device-only."""
    t = type(op)
    return t.perform is not Op.perform and t.lower is Op.lower


OP_REGISTRY: dict[str, type] = {}


def register_op(cls):
    OP_REGISTRY[cls.name] = cls
    return cls


def op_from_payload(name, payload, decode_graph=None):
    if name not in OP_REGISTRY:
        raise TypeMismatch(f"unknown op {name!r} in graph document")
    return OP_REGISTRY[name].from_payload(payload, decode_graph)


def broadcast_pattern(patterns) -> tuple:
    """Right-aligned broadcast: a dim is guaranteed-1 only if it is so (or
    absent) in every pattern (reference ``ops/base.py:117-129``)."""
    patterns = [tuple(p) for p in patterns]
    nd = max((len(p) for p in patterns), default=0)
    padded = [(True,) * (nd - len(p)) + p for p in patterns]
    return tuple(all(p[i] for p in padded) for i in range(nd))


def broadcast_shapes_checked(node, shapes) -> tuple:
    """Concrete broadcast with the reference's strictness: an extent-1 dim may
    stretch only where the input's type declares it broadcastable
    (reference ``ops/base.py:132-163``)."""
    shapes = [tuple(s) for s in shapes]
    nd = max((len(s) for s in shapes), default=0)
    out = [1] * nd
    for s in shapes:
        off = nd - len(s)
        for j, e in enumerate(s):
            i = j + off
            if e == 1:
                continue
            if out[i] == 1:
                out[i] = e
            elif out[i] != e:
                raise ShapeMismatch(f"{node.op.name}: incompatible extents {out[i]} and {e} at dim {i}")
    for x, s in zip(node.inputs, shapes):
        off = nd - len(s)
        for j, e in enumerate(s):
            if e == 1 and out[j + off] != 1 and not x.type.broadcastable[j]:
                raise ShapeMismatch(
                    f"{node.op.name}: {x!r} has runtime extent 1 at dim {j} where the type "
                    f"does not declare broadcastability (needs {out[j + off]})")
    return tuple(out)


# Name kept for drop-in code that imported it from the reference.
check_broadcast_shapes = broadcast_shapes_checked
