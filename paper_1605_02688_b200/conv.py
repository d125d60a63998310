"""2-d convolution on the device (reference ``ops/conv.py``
and the implementation-selection hook ``rewrites/convselect.py``).

Graph contract identical to the reference: an abstract placeholder op whose
``kind`` is forward / grad_inputs / grad_weights and whose ``algo`` is
chosen by the ``conv_select_implementation`` rewrite in stage
``abstract_select`` (``compile(conv_impl="gemm" | "reference" | "none")``);
NCHW data, KCHW filters, stride and zero-padding pairs, no flip, no
dilation; gradient kinds take the target's runtime shape vector.

Device lowering (the im2col -> tensor-core GEMM the reference's "gemm"
algorithm describes, ``ops/conv.py:108-157``):

  forward       cols = im2col(x)                 [N*Ho*Wo, C*kh*kw]
                outT = F[K, C*kh*kw] . cols^T     tx_gemm (tcgen05 TF32 for fp32)
                out  = outT viewed [N, K, Ho*Wo]  one strided copy (none if N == 1)
  grad_weights  dF   = dy^T[K, N*Ho*Wo] . cols
  grad_inputs   dcols = dy^T^T . F;  dx = col2im(dcols)  (deterministic gather)

``algo="reference"`` runs the same lowering with exact fp32 products
(CUDA-core GEMM) -- the debugging reference the reference keeps as direct
loops.
"""
from __future__ import annotations

import numpy as np

from .dtypes import is_float, promote
from .errors import AbstractOpRemaining, NotSupported, ShapeMismatch, TypeMismatch
from .graph import TensorType, Variable, apply
from .op import DISCONNECTED, UNKNOWN_SHAPE, Op, register_op
from .rewrite import register_rewrite
from .shaping import _shape_arg, shape_of

FORWARD, GRAD_INPUTS, GRAD_WEIGHTS = "forward", "grad_inputs", "grad_weights"
ABSTRACT, REFERENCE, GEMM = "abstract", "reference", "gemm"


def conv_output_size(size: int, kernel: int, stride: int, pad: int) -> int:
    out = (size + 2 * pad - kernel) // stride + 1
    if out <= 0:
        raise ShapeMismatch(f"convolution window {kernel} (pad {pad}) does not fit input extent {size}")
    return out


@register_op
class Conv2d(Op):
    """One member of the convolution trio, possibly still a placeholder."""

    name = "conv2d"
    foldable = False
    uses_values = True

    def __init__(self, kind: str, algo: str, stride=(1, 1), pad=(0, 0)):
        if kind not in (FORWARD, GRAD_INPUTS, GRAD_WEIGHTS):
            raise TypeMismatch(f"unknown conv kind {kind!r}")
        if algo not in (ABSTRACT, REFERENCE, GEMM):
            raise TypeMismatch(f"unknown conv algo {algo!r}")
        self.kind, self.algo = kind, algo
        self.stride = (int(stride[0]), int(stride[1]))
        self.pad = (int(pad[0]), int(pad[1]))

    @property
    def display_name(self):
        return f"conv2d.{self.kind}.{self.algo}"

    @property
    def is_abstract(self):
        return self.algo == ABSTRACT

    def attrs_key(self):
        return (self.kind, self.algo, self.stride, self.pad)

    def with_algo(self, algo: str) -> "Conv2d":
        return Conv2d(self.kind, algo, self.stride, self.pad)

    def infer_types(self, input_types):
        if self.kind == FORWARD:
            x, f = input_types
            if x.ndim != 4 or f.ndim != 4:
                raise TypeMismatch("conv2d expects rank-4 input and filters")
            return [TensorType(promote(x.dtype, f.dtype), (x.broadcastable[0], f.broadcastable[0], False, False))]
        a, dy, shp = input_types
        if a.ndim != 4 or dy.ndim != 4:
            raise TypeMismatch("conv2d gradient expects rank-4 operands")
        if shp.ndim != 1 or shp.dtype not in ("int32", "int64"):
            raise TypeMismatch("conv2d gradient expects an integer shape vector")
        return [TensorType(promote(a.dtype, dy.dtype), (False, False, False, False))]

    def check_runtime_shapes(self, node, shapes):
        if self.kind == FORWARD:
            x, f = shapes
            if x[1] != f[1]:
                raise ShapeMismatch(f"conv2d channel mismatch: input has {x[1]}, filters {f[1]}")

    def infer_shape(self, node, input_shapes, values=None):
        if self.kind == FORWARD:
            x, f = input_shapes
            if x is UNKNOWN_SHAPE or f is UNKNOWN_SHAPE:
                return [UNKNOWN_SHAPE]
            n, _, h, w = x
            k, _, kh, kw = f
            if None in (h, w, kh, kw):
                return [(n, k, None, None)]
            return [(n, k, conv_output_size(h, kh, self.stride[0], self.pad[0]),
                     conv_output_size(w, kw, self.stride[1], self.pad[1]))]
        dims = _shape_arg(node, 2, values)
        return [dims if dims is not None else (None, None, None, None)]

    def grad(self, inputs, output_grads):
        if self.kind != FORWARD:
            from .errors import NotDifferentiable
            raise NotDifferentiable(f"{self.display_name}: second-order convolution is not provided")
        x, f = inputs
        (v,) = output_grads
        gx = apply(Conv2d(GRAD_INPUTS, self.algo, self.stride, self.pad), [f, v, shape_of(x)])[0]
        gf = apply(Conv2d(GRAD_WEIGHTS, self.algo, self.stride, self.pad), [x, v, shape_of(f)])[0]
        return [gx if is_float(x.type.dtype) else DISCONNECTED, gf if is_float(f.type.dtype) else DISCONNECTED]

    def rop(self, inputs, input_perturbations):
        if self.kind != FORWARD:
            raise NotSupported(f"{self.display_name} has no R-operator rule")
        x, f = inputs
        dx, df = input_perturbations
        terms = []
        if dx is not None:
            terms.append(apply(Conv2d(FORWARD, self.algo, self.stride, self.pad), [dx, f])[0])
        if df is not None:
            terms.append(apply(Conv2d(FORWARD, self.algo, self.stride, self.pad), [x, df])[0])
        if not terms:
            return [None]
        return [terms[0] if len(terms) == 1 else terms[0] + terms[1]]

    def attrs_payload(self, encode_graph=None):
        return {"kind": self.kind, "algo": self.algo, "stride": list(self.stride), "pad": list(self.pad)}

    @classmethod
    def from_payload(cls, payload, decode_graph=None):
        return cls(payload["kind"], payload["algo"], payload["stride"], payload["pad"])

    # -- device lowering ---------------------------------------------------------
    def lower(self, node, plan):
        if self.is_abstract:
            raise AbstractOpRemaining(f"{self.display_name}: no convolution implementation was selected "
                                      "(compile with conv_impl='gemm' or 'reference')")
        from . import native
        mode = native.GEMM_SIMT if self.algo == REFERENCE else plan.fn.gemm_mode
        out = plan.layout(node.outputs[0])
        if out.numel == 0:
            return
        if self.kind == FORWARD:
            x, f = (plan.layout(v) for v in node.inputs)
            N, C, H, W = x.shape
            K, _, kh, kw = f.shape
            _, _, Ho, Wo = out.shape
            f = _contig(plan, f)
            if self._implicit_ok(mode, x.dtype, C, Wo):
                fr = plan.scratch((K, kh, kw, C), f.dtype)
                plan.emit_copy_layouts(plan.view_of(f, (K, kh, kw, C), (C * kh * kw, kw, 1, kh * kw), f.offset), fr)
                if out.contiguous():  # the epilogue stores NCHW directly
                    self._implicit(plan, x, self.pad, fr, out, kh, kw, var=node.inputs[0])
                    return
                res = plan.scratch((N * Ho * Wo, K), out.dtype)
                self._implicit(plan, x, self.pad, fr, res, kh, kw, var=node.inputs[0])
                plan.emit_copy_layouts(plan.view_of(res, (N, K, Ho * Wo), (Ho * Wo * K, 1, K), 0),
                                       plan.view_of(out, (N, K, Ho * Wo), (K * Ho * Wo, Ho * Wo, 1), out.offset))
                return
            cols = self._cols(plan, node.inputs[0], x, N * Ho * Wo, C * kh * kw, kh, kw)
            if self.algo == GEMM:
                # (u, v, c) patch order: the filters reordered to [K, kh, kw, C]
                fr = plan.scratch((K, kh, kw, C), f.dtype)
                plan.emit_copy_layouts(plan.view_of(f, (K, kh, kw, C), (C * kh * kw, kw, 1, kh * kw), f.offset), fr)
                f = fr
            fm = plan.view_of(f, (K, C * kh * kw), (C * kh * kw, 1), f.offset)
            colsT = plan.view_of(cols, (C * kh * kw, N * Ho * Wo), (1, C * kh * kw), 0)
            if N == 1:
                plan.emit_gemm(fm, colsT, plan.view_of(out, (K, Ho * Wo), (Ho * Wo, 1), out.offset), mode)
            else:
                outT = plan.scratch((K, N * Ho * Wo), out.dtype)
                plan.emit_gemm(fm, colsT, outT, mode)
                src = plan.view_of(outT, (N, K, Ho * Wo), (Ho * Wo, N * Ho * Wo, 1), 0)
                plan.emit_copy_layouts(src, plan.view_of(out, (N, K, Ho * Wo), (K * Ho * Wo, Ho * Wo, 1), out.offset))
            return
        a, dy = plan.layout(node.inputs[0]), plan.layout(node.inputs[1])
        N, K, Ho, Wo = dy.shape
        if (self.kind == GRAD_INPUTS and self.algo == GEMM and tuple(self.stride) == (1, 1)
                and self.pad[0] < a.shape[2] and self.pad[1] < a.shape[3]):
            # stride 1: the input gradient is the forward convolution of dy with
            # the flipped, channel-transposed filters (pad k-1-p): im2col of dy
            # and ONE GEMM straight into [N*H*W, C] -- no [N*Ho*Wo, C*kh*kw]
            # gradient-of-columns matrix and no gather over it (col2im was 324 us
            # of a 32x64x56x56 3x3 layer's step)
            f = _contig(plan, a)
            _, C, kh, kw = f.shape
            _, _, H, W = out.shape
            self._grad_inputs_as_conv(plan, f, _contig(plan, dy), out, N, K, C, H, W, kh, kw, mode)
            return
        dyT = plan.scratch((K, N * Ho * Wo), dy.dtype)
        plan.emit_copy_layouts(plan.view_of(dy, (K, N, Ho * Wo), (dy.strides[1], dy.strides[0], 1), dy.offset)
                               if dy.contiguous() else _contig(plan, dy, (K, N, Ho * Wo), (1, 0, 2)),
                               plan.view_of(dyT, (K, N, Ho * Wo), (N * Ho * Wo, Ho * Wo, 1), 0))
        if self.kind == GRAD_WEIGHTS:
            x = a
            _, C, kh, kw = out.shape
            cols = self._cols(plan, node.inputs[0], x, N * Ho * Wo, C * kh * kw, kh, kw)
            if self.algo == GEMM:  # (u, v, c) patch order: dW as [K, kh, kw, C], then to [K, C, kh, kw]
                gr = plan.scratch((K, kh, kw, C), out.dtype)
                plan.emit_gemm(dyT, plan.view_of(cols, (N * Ho * Wo, C * kh * kw), (C * kh * kw, 1), 0),
                               plan.view_of(gr, (K, C * kh * kw), (C * kh * kw, 1), 0), mode)
                plan.emit_copy_layouts(plan.view_of(gr, (K, C, kh, kw), (C * kh * kw, 1, kw * C, C), 0), out)
                return
            plan.emit_gemm(dyT, cols, plan.view_of(out, (K, C * kh * kw), (C * kh * kw, 1), out.offset), mode)
            return
        f = _contig(plan, a)
        _, C, kh, kw = f.shape
        _, _, H, W = out.shape
        dcols = plan.scratch((N * Ho * Wo, C * kh * kw), out.dtype)
        plan.emit_gemm(plan.view_of(dyT, (N * Ho * Wo, K), (1, N * Ho * Wo), 0),
                       plan.view_of(f, (K, C * kh * kw), (C * kh * kw, 1), f.offset), dcols, mode)
        win = self._win(kh, kw)
        lib = plan.lib
        dc, dx = plan.tx(dcols), plan.tx(out)

        def launch(stream):
            lib.check(lib.lib.tx_col2im(dc, dx, win, Ho, Wo, stream))
        plan.add_launch(launch)

    def _grad_inputs_as_conv(self, plan, f, dy4, out, N, K, C, H, W, kh, kw, mode):
        # fr[(u, v, k), c] = f[k, c, kh-1-u, kw-1-v]: a negative-stride view copied
        # contiguous, in the (u, v, k) patch order of the channel-contiguous dy
        fr = plan.scratch((kh, kw, K, C), out.dtype)
        plan.emit_copy_layouts(plan.view_of(f, (kh, kw, K, C), (-kw, -1, C * kh * kw, kh * kw),
                                            f.offset + (kh - 1) * kw + (kw - 1)), fr)
        ph, pw = kh - 1 - self.pad[0], kw - 1 - self.pad[1]
        Nn, Kk, Ho, Wo = dy4.shape
        if ph >= 0 and pw >= 0 and self._implicit_ok(mode, dy4.dtype, K, W):
            # filters as [C, (u, v, k)] rows for the implicit GEMM's K-major B
            frT = plan.scratch((C, kh, kw, K), out.dtype)
            plan.emit_copy_layouts(plan.view_of(fr, (C, kh, kw, K), (1, kw * K * C, K * C, C), 0), frT)
            if out.contiguous():  # the epilogue stores NCHW directly
                self._implicit(plan, dy4, (ph, pw), frT, out, kh, kw)
                return
            res = plan.scratch((N * H * W, C), out.dtype)
            self._implicit(plan, dy4, (ph, pw), frT, res, kh, kw)
            plan.emit_copy_layouts(plan.view_of(res, (N, C, H * W), (H * W * C, 1, C), 0),
                                   plan.view_of(out, (N, C, H * W), (C * H * W, H * W, 1), out.offset))
            return
        dyh = self._hwc(plan, None, dy4)
        cols = plan.scratch((N * H * W, K * kh * kw), out.dtype)
        lib = plan.lib
        win = (__import__("ctypes").c_int * 6)(kh, kw, 1, 1, ph, pw)
        td, tc = plan.tx(dyh), plan.tx(cols)

        def launch(stream):
            lib.check(lib.lib.tx_im2col_hwc(td, tc, win, stream))
        plan.add_launch(launch)
        # [N*H*W, kh*kw*K] . [kh*kw*K, C] -> [N*H*W, C], then to NCHW
        res = plan.scratch((N * H * W, C), out.dtype)
        plan.emit_gemm(cols, plan.view_of(fr, (K * kh * kw, C), (C, 1), 0), res, mode)
        plan.emit_copy_layouts(plan.view_of(res, (N, C, H * W), (H * W * C, 1, C), 0),
                               plan.view_of(out, (N, C, H * W), (C * H * W, H * W, 1), out.offset))

    def _implicit_ok(self, mode, dtype, C, Wo) -> bool:
        """The tensor-core implicit GEMM (tx_conv_implicit) applies: GEMM
        algorithm at TF32, stride 1, float32, 32-channel blocks, output rows
        of at most 128 pixels."""
        from . import native
        return (self.algo == GEMM and mode in (native.GEMM_AUTO, native.GEMM_TC) and tuple(self.stride) == (1, 1)
                and dtype == "float32" and C % 32 == 0 and 0 < Wo <= 128 and not _NO_IMPLICIT)

    def _implicit(self, plan, x, pad, wr, res, kh, kw, var=None):
        """res = conv(x, w) with x [N, C, H, W] (any strides), wr [K, kh, kw,
        C] contiguous, res [N*P*Q, K] or [N, K, P, Q] contiguous: x goes to a
        zero-padded NHWC buffer (memset + one strided copy), then ONE
        tcgen05 launch reads it through 4-D TMA boxes per (tap, channel
        block) -- no patch matrix (the explicit form wrote and re-read
        N*P*Q*kh*kw*C floats: 231 MB for a 32x64x56x56 3x3 layer)."""
        N, C, H, W = x.shape
        ph, pw = pad
        Hp, Wp = H + 2 * ph, W + 2 * pw
        xp = self._padded_nhwc(plan, var, x, pad)
        K = wr.shape[0]
        lib = plan.lib
        tx_ = plan.tx(xp)
        tw = plan.tx(wr, (K, kh * kw * C), (kh * kw * C, 1))
        tr = plan.tx(res)
        win = (__import__("ctypes").c_int * 2)(kh, kw)

        def launch(stream):
            lib.check(lib.lib.tx_conv_implicit(tx_, tw, tr, win, stream))
        plan.add_launch(launch)

    def _padded_nhwc(self, plan, var, x, pad):
        """Zero-padded NHWC copy of ``x`` ([N, Hp, Wp, C]), built once per step
        plan per (variable, padding): the layer's weight gradient gathers its
        patch matrix from the same buffer (see ``_cols``)."""
        N, C, H, W = x.shape
        ph, pw = pad
        Hp, Wp = H + 2 * ph, W + 2 * pw
        cache = plan.__dict__.setdefault("_xpad_cache", {})
        key = None if var is None else (var.id, x.shape, x.strides, ph, pw)
        if key is not None and key in cache:
            return cache[key]
        xp = plan.scratch((N, Hp, Wp, C), x.dtype)
        lib = plan.lib
        tx_, tp = plan.tx(x), plan.tx(xp)
        pads = (__import__("ctypes").c_int * 2)(ph, pw)

        def launch(stream):  # one pass: transposed interior + zero borders
            lib.check(lib.lib.tx_pad_nhwc(tx_, tp, pads, stream))
        plan.add_launch(launch)
        if key is not None:
            cache[key] = xp
        return xp

    def _win(self, kh, kw):
        import ctypes
        return (ctypes.c_int * 6)(kh, kw, self.stride[0], self.stride[1], self.pad[0], self.pad[1])

    def _cols(self, plan, var, x, rows, ckk, kh, kw):
        """The patch matrix of variable ``var`` (layout ``x``) for this window,
        built once per step plan: a layer's forward and its weight gradient
        read the same matrix (``var`` is live until the later of the two, so
        its buffer is unchanged; keyed on the variable, not the address, which
        the arena may hand to another tensor once ``var`` is dead)."""
        cache = plan.__dict__.setdefault("_im2col_cache", {})
        hwc = self.algo == GEMM
        key = (var.id, x.shape, x.strides, kh, kw, tuple(self.stride), tuple(self.pad), hwc)
        cols = cache.get(key)
        if cols is None:
            cols = plan.scratch((rows, ckk), x.dtype)
            if hwc:
                # (u, v, c) columns from a channel-contiguous copy of x: every
                # gather and store runs along c, 128-bit (r02: the (c, u, v)
                # gather over NCHW was L1-wavefront bound at 91 us for 231 MB);
                # the forward's zero-padded NHWC copy when the implicit GEMM
                # built one (window padding 0 over it: the same columns)
                xp = plan.__dict__.get("_xpad_cache", {}).get((var.id, x.shape, x.strides, self.pad[0], self.pad[1]))
                lib, win = plan.lib, self._win(kh, kw)
                if xp is not None:
                    N_, Hp, Wp, C_ = xp.shape
                    xh = plan.view_of(xp, (N_, C_, Hp, Wp), (Hp * Wp * C_, 1, Wp * C_, C_), 0)
                    win = (__import__("ctypes").c_int * 6)(kh, kw, self.stride[0], self.stride[1], 0, 0)
                else:
                    xh = self._hwc(plan, var, x)
                tx_, tc = plan.tx(xh), plan.tx(cols)

                def launch(stream):
                    lib.check(lib.lib.tx_im2col_hwc(tx_, tc, win, stream))
                plan.add_launch(launch)
            else:
                self._im2col(plan, x, cols, kh, kw)
            cache[key] = cols
        return cols

    def _hwc(self, plan, var, x):
        """[N, C, H, W] view of a channel-contiguous (NHWC) copy of ``x`` (x
        itself when its channel stride is already 1)."""
        if x.strides[1] == 1:
            return x
        N, C, H, W = x.shape
        dst = plan.scratch((N, H, W, C), x.dtype)
        plan.emit_copy_layouts(plan.view_of(x, (N, H, W, C), (x.strides[0], x.strides[2], x.strides[3], x.strides[1]),
                                            x.offset), dst)
        return plan.view_of(dst, (N, C, H, W), (H * W * C, 1, W * C, C), 0)

    def _im2col(self, plan, x, cols, kh, kw):
        lib = plan.lib
        win = self._win(kh, kw)
        tx, tc = plan.tx(x), plan.tx(cols)

        def launch(stream):
            lib.check(lib.lib.tx_im2col(tx, tc, win, stream))
        plan.add_launch(launch)


_NO_IMPLICIT = bool(__import__("os").environ.get("TX_CONV_NO_IMPLICIT"))  # A/B: explicit im2col for every conv


def _contig(plan, lay, shape=None, perm=None):
    if shape is None:
        if lay.contiguous():
            return lay
        dst = plan.scratch(lay.shape, lay.dtype)
        plan.emit_copy_layouts(lay, dst)
        return dst
    # general (non-contiguous dy): make it contiguous first, then view with the permutation
    c = _contig(plan, lay)
    st = (c.strides[1], c.strides[0], 1)
    return plan.view_of(c, shape, st, c.offset)


def conv2d(x: Variable, filters: Variable, stride=(1, 1), pad=(0, 0)) -> Variable:
    """Abstract 2-d cross-correlation; the implementation is chosen at compile
    time (``conv_impl``)."""
    return apply(Conv2d(FORWARD, ABSTRACT, stride, pad), [x, filters])[0]


@register_rewrite("conv_select_implementation", "abstract_select", "global")
def conv_select_implementation(fgraph, ctx, emit) -> int:
    """Replace every placeholder with the implementation ``ctx.conv_impl``
    asks for (gemm by default; "none" leaves placeholders, which fails at
    execution) -- reference ``rewrites/convselect.py:10-33``."""
    if ctx.conv_impl == "none":
        return 0
    algo = GEMM if ctx.conv_impl == "gemm" else REFERENCE
    applied = 0
    for node in fgraph.toposort():
        if node.id not in fgraph.nodes or not (isinstance(node.op, Conv2d) and node.op.is_abstract):
            continue
        outs = apply(node.op.with_algo(algo), node.inputs)
        fgraph.replace_all(list(zip(node.outputs, outs)), "conv_select_implementation")
        emit(node=node, replaced=node.op.display_name, replacement=outs[0].owner.op.display_name)
        applied += 1
    return applied
