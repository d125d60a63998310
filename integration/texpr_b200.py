"""The reference-side binding: the B200 library as a plugin of the REFERENCE's
own runtime (the module a texpr maintainer would add as ``texpr/b200.py``).

Pure ctypes + NumPy over the C ABI of ``include/texpr_b200.h`` -- no torch,
no import of this repo's Python package -- so it shows exactly what the
reference's FFI for this path binds.  It uses the reference's two plugin
hooks:

* an operator registered with ``@register_op`` (reference ``ops/base.py:100-111``)
  whose ``perform`` (the reference's host-array contract, ``Dot.perform``
  ``ops/linalg.py:42-62``) runs ``tx_gemm`` on the B200: H2D of the two
  operands, the tcgen05 GEMM, D2H of the product;
* a local rewrite in stage ``abstract_select`` (``rewrites/engine.py:26``, the
  stage the reference uses to swap implementations, ``rewrites/convselect.py``)
  that replaces every rank-2 float32 ``Dot`` with that op.

``install(texpr, lib_path, precision)`` registers both into the given texpr
module; the rewrite carries the tag "b200", so a user opts in per compile with
``include=("b200_select_dot",)``.  Precision: "3xtf32" (default; fp32-sgemm
class, what the reference computes) or "tf32".
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

MAX_RANK = 8
TX_F32 = 0
GEMM_MODE = {"tf32": 0, "3xtf32": 3}


class TxTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("shape", ctypes.c_int64 * MAX_RANK), ("strides", ctypes.c_int64 * MAX_RANK)]


def _tensor(ptr, shape, strides):
    t = TxTensor()
    t.data, t.dtype, t.ndim = ptr, TX_F32, len(shape)
    for i, (s, st) in enumerate(zip(shape, strides)):
        t.shape[i], t.strides[i] = int(s), int(st)
    return t


class B200:
    """The handful of C entry points a Dot plugin needs."""

    def __init__(self, path):
        L = ctypes.CDLL(path)
        vp, sz, P = ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER
        L.tx_last_error.restype = ctypes.c_char_p
        for name, args in {"tx_init": [ctypes.c_int], "tx_device_alloc": [sz, P(vp)], "tx_device_free": [vp],
                           "tx_memcpy_async": [vp, vp, sz, ctypes.c_int, vp], "tx_stream_sync": [vp],
                           "tx_gemm_workspace": [P(TxTensor)] * 3 + [ctypes.c_int, P(sz)],
                           "tx_gemm": [P(TxTensor)] * 3 + [vp, ctypes.c_int, vp, sz, vp]}.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
        self.L = L
        self.check(L.tx_init(0))
        self.calls = 0

    def check(self, rc):
        if rc:
            raise RuntimeError(f"tx error {rc}: {self.L.tx_last_error().decode()}")

    def gemm(self, a: np.ndarray, b: np.ndarray, mode: int) -> np.ndarray:
        """C = A . B for float32 host matrices on the B200 (any strides: the
        operands are staged contiguous)."""
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        (M, K), (_, N) = a.shape, b.shape
        c = np.empty((M, N), np.float32)
        L, ptrs = self.L, []
        try:
            def dev(nbytes):
                p = ctypes.c_void_p()
                self.check(L.tx_device_alloc(nbytes, ctypes.byref(p)))
                ptrs.append(p.value)
                return p.value
            da, db, dc = dev(a.nbytes), dev(b.nbytes), dev(c.nbytes)
            A, B, C = _tensor(da, (M, K), (K, 1)), _tensor(db, (K, N), (N, 1)), _tensor(dc, (M, N), (N, 1))
            wsb = ctypes.c_size_t()
            self.check(L.tx_gemm_workspace(ctypes.byref(A), ctypes.byref(B), ctypes.byref(C), mode, ctypes.byref(wsb)))
            ws = dev(wsb.value) if wsb.value else None
            self.check(L.tx_memcpy_async(da, a.ctypes.data, a.nbytes, 0, None))
            self.check(L.tx_memcpy_async(db, b.ctypes.data, b.nbytes, 0, None))
            self.check(L.tx_gemm(ctypes.byref(A), ctypes.byref(B), ctypes.byref(C), None, mode, ws, wsb.value, None))
            self.check(L.tx_memcpy_async(c.ctypes.data, dc, c.nbytes, 1, None))
            self.check(L.tx_stream_sync(None))
        finally:
            for p in ptrs:
                L.tx_device_free(p)
        self.calls += 1
        return c


def install(texpr, lib_path=None, precision="3xtf32"):
    """Register the B200 Dot op and its selection rewrite into ``texpr``."""
    from texpr.graph import apply
    from texpr.ops.base import register_op
    from texpr.ops.linalg import Dot
    from texpr.rewrites.engine import register_rewrite
    lib = B200(lib_path or os.environ.get("TEXPR_B200_LIB", "libtexpr_b200.so"))
    mode = GEMM_MODE[precision]

    @register_op
    class B200Dot(Dot):
        """``Dot`` whose perform runs tx_gemm (same types, shapes, gradient)."""
        name = "b200_dot"

        def perform(self, inputs, output_buffers=None):
            a, b = inputs
            return [lib.gemm(a, b, mode)]

    def select_dot(fgraph, node, ctx):
        op = node.op
        if type(op) is not Dot:
            return None
        a, b = node.inputs
        if a.type.ndim != 2 or b.type.ndim != 2 or a.type.dtype != "float32" or b.type.dtype != "float32":
            return None
        return [(node.outputs[0], apply(B200Dot(), [a, b])[0])]

    register_rewrite("b200_select_dot", "abstract_select", "local", tags=("b200",))(select_dot)
    return lib, B200Dot
