"""Dot: rank-1/2 inner products (reference ``ops/linalg.py:13-123``).

Lowered to ``tx_gemm``: operand transposes arrive as strides (DimShuffle
views), and the native dispatcher chooses the tcgen05/TMEM TF32 tensor-core
kernel for large fp32 problems, a memory-bound skinny kernel when one of
M/N/K is tiny (the ``[B,10]`` softmax layers), and a SIMT kernel for float64.
"""
from __future__ import annotations

from .dtypes import is_float, promote
from .errors import ShapeMismatch, TypeMismatch
from .graph import TensorType, Variable, apply
from .op import DISCONNECTED, UNKNOWN_SHAPE, Op, register_op
from .shaping import dimshuffle


@register_op
class Dot(Op):
    name = "dot"

    def infer_types(self, input_types):
        a, b = input_types
        if a.ndim not in (1, 2) or b.ndim not in (1, 2):
            raise TypeMismatch(f"dot expects rank 1 or 2 operands, got {a.ndim} and {b.ndim}")
        if a.ndim == 2 and b.ndim == 2:
            bc = (a.broadcastable[0], b.broadcastable[1])
        elif a.ndim == 2:
            bc = (a.broadcastable[0],)
        elif b.ndim == 2:
            bc = (b.broadcastable[1],)
        else:
            bc = ()
        return [TensorType(promote(a.dtype, b.dtype), bc)]

    def check_runtime_shapes(self, node, shapes):
        a, b = shapes
        ka = a[-1]
        kb = b[0] if len(b) >= 1 else 1
        if ka != kb:
            raise ShapeMismatch(f"dot: inner dimensions disagree ({tuple(a)} vs {tuple(b)})")

    def infer_shape(self, node, input_shapes):
        a, b = input_shapes
        if a is UNKNOWN_SHAPE or b is UNKNOWN_SHAPE:
            return [UNKNOWN_SHAPE]
        an, bn = len(a), len(b)
        if an == 2 and bn == 2:
            return [(a[0], b[1])]
        if an == 2:
            return [(a[0],)]
        if bn == 2:
            return [(b[1],)]
        return [()]

    def grad(self, inputs, output_grads):
        from .elemwise import sum_to_matching_shape
        (a, b), (v,) = inputs, output_grads
        an, bn = a.type.ndim, b.type.ndim
        if an == 2 and bn == 2:
            ga, gb = dot(v, dimshuffle(b, (1, 0))), dot(dimshuffle(a, (1, 0)), v)
        elif an == 2:
            ga = dimshuffle(v, (0, "x")) * dimshuffle(b, ("x", 0))
            gb = dot(dimshuffle(a, (1, 0)), v)
        elif bn == 2:
            ga = dot(b, v)
            gb = dimshuffle(a, (0, "x")) * dimshuffle(v, ("x", 0))
        else:
            ga, gb = v * b, v * a
        return [DISCONNECTED if not is_float(x.type.dtype) else sum_to_matching_shape(g, x)
                for x, g in ((a, ga), (b, gb))]

    def rop(self, inputs, input_perturbations):
        (a, b), (da, db) = inputs, input_perturbations
        terms = ([dot(da, b)] if da is not None else []) + ([dot(a, db)] if db is not None else [])
        if not terms:
            return [None]
        return [terms[0] if len(terms) == 1 else terms[0] + terms[1]]

    def fold(self, values):
        import numpy as np
        a, b = values
        if a.size * b.size > 1 << 16:
            return None
        return [np.asarray(np.dot(a, b))]

    def lower(self, node, plan):
        plan.emit_dot(node)


def dot(a: Variable, b: Variable) -> Variable:
    return apply(Dot(), [a, b])[0]


# epilogue kinds (include/texpr_b200.h TX_EPI_*)
EPI_BIAS, EPI_BIAS_TANH, EPI_MUL_1MSQR, EPI_BIAS_TANH_DUAL, EPI_MUL_AUX, EPI_SGD = 1, 2, 3, 4, 5, 6
EPI_ADD_AUX_BIAS = 7
_EPI_NAMES = {EPI_BIAS: "bias", EPI_BIAS_TANH: "bias_tanh", EPI_MUL_1MSQR: "mul_1msqr",
              EPI_BIAS_TANH_DUAL: "bias_tanh_dual", EPI_MUL_AUX: "mul_aux", EPI_SGD: "sgd",
              EPI_ADD_AUX_BIAS: "add_aux_bias"}


@register_op
class DotEpilogue(Op):
    """dot(a, b) with its elementwise consumer folded into the GEMM epilogue.

    Produced only by the ``fuse_gemm_epilogue`` rewrite (``fusion.py``) after
    differentiation; inputs are (a, b, aux) and the outputs are exactly the
    replaced consumer's outputs, computed with the same scalar ops in the
    same order (see ``Epi`` in ``csrc/tx_gemm.h``):
      bias            out = aux[n] + a.b
      bias_tanh       out = tanh(aux[n] + a.b)
      mul_1msqr       out = (a.b) * (1 - aux^2)      (aux = the forward's h)
      bias_tanh_dual  out = tanh(aux[n] + a.b), out2 = 1 - out^2
      mul_aux         out = (a.b) * aux
      sgd             out = aux - alpha * (a.b)      (a weight's SGD update from its gradient GEMM;
                                                      the output may be written in place over aux)
      add_aux_bias    out = bias[n] + (aux + a.b)    (inputs a, b, aux, bias: a recurrent
                                                      pre-activation with its input projection)
    """

    name = "dot_epilogue"
    has_grad = False
    gemm_operands = True

    @property
    def elementwise_in_place(self):
        return self.kind == EPI_SGD

    def __init__(self, kind: int, alpha: float = 0.0, alpha_dtype: str = "float32"):
        self.kind = int(kind)
        self.alpha = float(alpha)
        self.alpha_dtype = alpha_dtype

    @property
    def display_name(self):
        return f"dot+{_EPI_NAMES.get(self.kind, self.kind)}"

    def attrs_key(self):
        return (self.kind, self.alpha, self.alpha_dtype)

    def infer_types(self, input_types):
        a, b, aux = input_types[:3]
        (t,) = Dot().infer_types([a, b])
        if self.kind == EPI_BIAS_TANH_DUAL:
            return [t, t]
        return [t]

    def check_runtime_shapes(self, node, shapes):
        Dot().check_runtime_shapes(node, shapes[:2])
        # the replaced elementwise node's broadcast check (reference
        # ops/base.py:132-163): a bias must match the product's last axis,
        # an [M,N] operand its shape
        (out,) = Dot().infer_shape(node, shapes[:2])[:1]
        aux = tuple(shapes[2])
        if self.kind in (EPI_BIAS, EPI_BIAS_TANH, EPI_BIAS_TANH_DUAL):
            ok = len(aux) >= 1 and aux[-1] == out[-1] and all(d == 1 for d in aux[:-1])
        else:
            ok = aux == tuple(out)
        if ok and self.kind == EPI_ADD_AUX_BIAS:
            bias = tuple(shapes[3])
            ok = len(bias) >= 1 and bias[-1] == out[-1] and all(d == 1 for d in bias[:-1])
        if not ok:
            raise ShapeMismatch(f"{self.display_name}: operand shape {aux} does not broadcast to {tuple(out)}")

    def infer_shape(self, node, input_shapes):
        (s,) = Dot().infer_shape(node, input_shapes[:2])
        return [s, s] if self.kind == EPI_BIAS_TANH_DUAL else [s]

    def grad(self, inputs, output_grads):
        from .errors import NotDifferentiable
        raise NotDifferentiable("dot_epilogue is created after differentiation")

    def expand(self, inputs):
        """The reference-op form (``dot`` + ``elemwise``) of this node, with the
        same scalar operations in the same order as the epilogue -- used to
        save portable graphs (``serialize.portable_outputs``)."""
        from .elemwise import make
        a, b, aux = inputs[:3]
        z = dot(a, b)
        if self.kind == EPI_ADD_AUX_BIAS:
            return [make("add", [inputs[3], make("add", [aux, z])])]
        if self.kind == EPI_BIAS:
            return [make("add", [aux, z])]
        if self.kind == EPI_BIAS_TANH:
            return [make("tanh", [make("add", [aux, z])])]
        if self.kind == EPI_MUL_1MSQR:
            return [make("mul", [z, make("sub", [1.0, make("sqr", [aux])])])]
        if self.kind == EPI_BIAS_TANH_DUAL:
            h = make("tanh", [make("add", [aux, z])])
            return [h, make("sub", [1.0, make("sqr", [h])])]
        if self.kind == EPI_MUL_AUX:
            return [make("mul", [z, aux])]
        if self.kind == EPI_SGD:
            from .graph import Constant
            return [make("sub", [aux, make("mul", [Constant(self.alpha, dtype=self.alpha_dtype), z])])]
        raise NotImplementedError(f"epilogue kind {self.kind}")

    def lower(self, node, plan):
        from . import native
        epi = native.TxEpilogue()
        epi.kind = self.kind
        epi.aux = plan.tx(node.inputs[2])
        epi.alpha = self.alpha
        if self.kind == EPI_ADD_AUX_BIAS:
            epi.aux2 = plan.tx(node.inputs[3])
        if self.kind == EPI_BIAS_TANH_DUAL:
            epi.out2 = plan.tx(node.outputs[1])
        plan.emit_dot(node, epilogue=epi)

    def attrs_payload(self, encode_graph=None):
        return {"kind": self.kind, "alpha": self.alpha, "alpha_dtype": self.alpha_dtype}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["kind"], payload.get("alpha", 0.0), payload.get("alpha_dtype", "float32"))


@register_op
class NarrowLayerGrad(Op):
    """The backward of a tanh layer ``h`` feeding a narrow dense layer
    (``z = h.W + b``, z of width k <= 16), fused into one pass over h.

    Produced only by the ``fuse_gemm_epilogue`` rewrite (``fusion.py``) from
    nodes the differentiated graph already holds (reference Dot.grad
    ``ops/linalg.py:68-70``, the tanh-grad composite, the bias gradient's
    ``Sum[0]`` from ``sum_to_matching_shape`` ``ops/elemwise.py:411-442``).
    Inputs (dz, wt, h[, w]); outputs, with the replaced nodes' rounding:
      dh = dot(dz, wt) * (1 - h^2)        the dot+mul_1msqr node
      gW = dot(h^T, dz)                   or, with ``sgd``, w - alpha * dot(h^T, dz)
      db = sum(dh, axis=0)                only with ``with_db``
    Lowered to ``tx_narrow_grad`` (``csrc/tx_narrow.cu``).
    """

    name = "narrow_grad"
    has_grad = False
    # the SGD output is written element by element in a second kernel after
    # every read of w (and of its transposed view wt): in-place safe
    elementwise_in_place = True
    reads_before_writes = True

    def __init__(self, sgd: bool = False, alpha: float = 0.0, alpha_dtype: str = "float32", with_db: bool = False):
        self.sgd = bool(sgd)
        self.alpha = float(alpha)
        self.alpha_dtype = alpha_dtype
        self.with_db = bool(with_db)

    @property
    def display_name(self):
        return "narrow_grad" + ("+sgd" if self.sgd else "") + ("+db" if self.with_db else "")

    def attrs_key(self):
        return (self.sgd, self.alpha, self.alpha_dtype, self.with_db)

    def infer_types(self, input_types):
        dz, wt, h = input_types[:3]
        (t_dh,) = Dot().infer_types([dz, wt])
        t_gw = TensorType(t_dh.dtype, (h.broadcastable[1], dz.broadcastable[1]))
        out = [t_dh, t_gw]
        if self.with_db:
            out.append(TensorType(t_dh.dtype, (t_dh.broadcastable[1],)))
        return out

    def check_runtime_shapes(self, node, shapes):
        dz, wt, h = shapes[:3]
        Dot().check_runtime_shapes(node, [dz, wt])
        if tuple(h) != (dz[0], wt[1]):
            raise ShapeMismatch(f"narrow_grad: h {tuple(h)} does not match dot(dz, wt) {(dz[0], wt[1])}")
        if self.sgd and tuple(shapes[3]) != (h[1], dz[1]):
            raise ShapeMismatch("narrow_grad: updated weight shape differs from the gradient's")

    def infer_shape(self, node, input_shapes):
        dz, wt, h = input_shapes[:3]
        if UNKNOWN_SHAPE in (dz, wt, h):
            return [UNKNOWN_SHAPE] * len(node.outputs)
        out = [(dz[0], wt[1]), (h[1], dz[1])]
        if self.with_db:
            out.append((wt[1],))
        return out

    def grad(self, inputs, output_grads):
        from .errors import NotDifferentiable
        raise NotDifferentiable("narrow_grad is created after differentiation")

    def shard_rule(self, states, sharded, partial, replicated):
        """Data-parallel states: batch rows sharded, weights replicated ->
        dh row-sharded, gW and db partial sums."""
        dz, wt, h = states[:3]
        if dz != sharded(0) or h != sharded(0) or wt != replicated or (self.sgd and states[3] != replicated):
            return None
        if self.sgd:
            return None  # an update from a partial sum needs the allreduce first
        return [sharded(0), partial] + ([partial] if self.with_db else [])

    def expand(self, inputs):
        """Reference-op form (dot, elemwise, sum) with the same scalar ops."""
        from .elemwise import make
        from .reduce import Sum
        dz, wt, h = inputs[:3]
        dh = make("mul", [dot(dz, wt), make("sub", [1.0, make("sqr", [h])])])
        gw = dot(dimshuffle(h, (1, 0)), dz)
        if self.sgd:
            from .graph import Constant
            gw = make("sub", [inputs[3], make("mul", [Constant(self.alpha, dtype=self.alpha_dtype), gw])])
        out = [dh, gw]
        if self.with_db:
            out.append(apply(Sum((0,)), [dh])[0])
        return out

    def workspace_bytes(self, plan, node):
        return plan.lib.narrow_grad_workspace(*self._tensors(plan, node, noptr=True), plan.fn.gemm_mode)

    def _tensors(self, plan, node, noptr=False):
        from . import native
        mk = plan._tx_noptr if noptr else plan.tx
        lay = plan.layout
        dz, wt, h = (mk(lay(v)) for v in node.inputs[:3])
        dh, gw = mk(lay(node.outputs[0])), mk(lay(node.outputs[1]))
        db = mk(lay(node.outputs[2])) if self.with_db else native.TxTensor()
        return dz, wt, h, dh, gw, db

    def lower(self, node, plan):
        from . import native
        dz, wt, h, dh, gw, db = self._tensors(plan, node)
        epi = native.TxEpilogue()
        if self.sgd:
            epi.kind = native.EPI_SGD
            epi.aux = plan.tx(node.inputs[3])
            epi.alpha = self.alpha
        ws, wsb = plan.workspace(node)
        mode = plan.fn.gemm_mode
        lib = plan.lib
        f = lib.lib.tx_narrow_grad

        def launch(stream):
            lib.check(f(dz, wt, h, dh, gw, epi, db, mode, ws, wsb, stream))
        plan.add_launch(launch)

    def attrs_payload(self, encode_graph=None):
        return {"sgd": self.sgd, "alpha": self.alpha, "alpha_dtype": self.alpha_dtype, "with_db": self.with_db}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["sgd"], payload["alpha"], payload["alpha_dtype"], payload["with_db"])
