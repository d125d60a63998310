"""ctypes binding of ``libtexpr_b200.so`` (C ABI: ``include/texpr_b200.h``).

This is the only path from Python to the device.  If the library is missing
or no GPU is present every compute entry point raises — there is no host
fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .dtypes import DTYPE_CODE
from .errors import DeviceError, NotSupported

MAX_RANK = 8
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtexpr_b200.so")

EXPORTS = [
    "tx_version", "tx_last_error", "tx_init", "tx_device_info", "tx_stream_create", "tx_stream_destroy",
    "tx_stream_sync", "tx_event_create", "tx_event_destroy", "tx_event_record", "tx_stream_wait_event",
    "tx_event_elapsed_ms", "tx_event_sync", "tx_memcpy_async", "tx_memset_async", "tx_host_register", "tx_host_unregister",
    "tx_device_alloc", "tx_device_free",
    "tx_graph_begin", "tx_graph_end", "tx_graph_launch", "tx_graph_destroy", "tx_copy",
    "tx_ew_compile", "tx_ew_check", "tx_ew_launch", "tx_ew_destroy",
    "tx_kernel_compile", "tx_kernel_launch", "tx_kernel_destroy",
    "tx_reduce_workspace", "tx_reduce", "tx_check_values", "tx_im2col", "tx_im2col_hwc", "tx_col2im", "tx_conv_implicit", "tx_pad_nhwc",
    "tx_gemm_workspace", "tx_gemm", "tx_gemm_path", "tx_narrow_grad_workspace", "tx_narrow_grad",
    "tx_nccl_unique_id", "tx_nccl_init", "tx_nccl_allreduce_sum", "tx_nccl_destroy",
]


class TxTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("shape", ctypes.c_int64 * MAX_RANK), ("strides", ctypes.c_int64 * MAX_RANK)]


class TxEpilogue(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("aux", TxTensor), ("out2", TxTensor), ("alpha", ctypes.c_double),
                ("aux2", TxTensor)]


EPI_NONE, EPI_BIAS, EPI_BIAS_TANH, EPI_MUL_1MSQR, EPI_BIAS_TANH_DUAL, EPI_MUL_AUX, EPI_SGD = 0, 1, 2, 3, 4, 5, 6
EPI_ADD_AUX_BIAS = 7
GEMM_AUTO, GEMM_SIMT, GEMM_TC, GEMM_3XTF32 = 0, 1, 2, 3


def make_tensor(ptr: int, dtype: str, shape, strides) -> TxTensor:
    t = TxTensor()
    t.data = ptr
    t.dtype = DTYPE_CODE[dtype]
    t.ndim = len(shape)
    for i, (s, st) in enumerate(zip(shape, strides)):
        t.shape[i] = int(s)
        t.strides[i] = int(st)
    return t


class Library:
    """Thin wrapper: every call checks the status and raises DeviceError."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise NotSupported(f"native library not built: {path} (run __graft_entry__.build())")
        self.path = path
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.tx_last_error.restype = ctypes.c_char_p
        vp, sz, i64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int64
        P = ctypes.POINTER
        sig = {
            "tx_init": [ctypes.c_int],
            "tx_device_info": [P(ctypes.c_int), P(ctypes.c_int), P(ctypes.c_int), P(i64)],
            "tx_stream_create": [P(vp)], "tx_stream_destroy": [vp], "tx_stream_sync": [vp],
            "tx_event_create": [P(vp)], "tx_event_destroy": [vp], "tx_event_record": [vp, vp],
            "tx_stream_wait_event": [vp, vp], "tx_event_elapsed_ms": [vp, vp, P(ctypes.c_float)],
            "tx_event_sync": [vp],
            "tx_memcpy_async": [vp, vp, sz, ctypes.c_int, vp], "tx_memset_async": [vp, ctypes.c_int, sz, vp],
            "tx_host_register": [vp, sz], "tx_host_unregister": [vp],
            "tx_device_alloc": [sz, P(vp)], "tx_device_free": [vp],
            "tx_graph_begin": [vp], "tx_graph_end": [vp, P(vp)], "tx_graph_launch": [vp, vp],
            "tx_graph_destroy": [vp], "tx_copy": [P(TxTensor), P(TxTensor), vp],
            "tx_ew_compile": [ctypes.c_char_p, ctypes.c_char_p, P(vp)],
            "tx_ew_check": [ctypes.c_char_p, ctypes.c_char_p, P(sz)],
            "tx_ew_launch": [vp, ctypes.c_int, ctypes.c_int, P(TxTensor), vp, vp], "tx_ew_destroy": [vp],
            "tx_kernel_compile": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, P(vp)],
            "tx_kernel_launch": [vp, ctypes.c_uint, ctypes.c_uint, vp, vp], "tx_kernel_destroy": [vp],
            "tx_reduce_workspace": [ctypes.c_int, P(TxTensor), ctypes.c_uint32, P(sz)],
            "tx_check_values": [P(TxTensor), vp, ctypes.c_int, ctypes.c_int, ctypes.c_double, vp],
            "tx_im2col": [P(TxTensor), P(TxTensor), P(ctypes.c_int), vp],
            "tx_im2col_hwc": [P(TxTensor), P(TxTensor), P(ctypes.c_int), vp],
            "tx_conv_implicit": [P(TxTensor), P(TxTensor), P(TxTensor), P(ctypes.c_int), vp],
            "tx_pad_nhwc": [P(TxTensor), P(TxTensor), P(ctypes.c_int), vp],
            "tx_col2im": [P(TxTensor), P(TxTensor), P(ctypes.c_int), i64, i64, vp],
            "tx_reduce": [ctypes.c_int, P(TxTensor), ctypes.c_uint32, P(TxTensor), vp, sz, vp],
            "tx_gemm_workspace": [P(TxTensor), P(TxTensor), P(TxTensor), ctypes.c_int, P(sz)],
            "tx_gemm": [P(TxTensor), P(TxTensor), P(TxTensor), P(TxEpilogue), ctypes.c_int, vp, sz, vp],
            "tx_gemm_path": [P(TxTensor), P(TxTensor), P(TxTensor), ctypes.c_int, P(ctypes.c_int)],
            "tx_narrow_grad_workspace": [P(TxTensor)] * 6 + [ctypes.c_int, P(sz)],
            "tx_narrow_grad": [P(TxTensor)] * 5 + [P(TxEpilogue), P(TxTensor), ctypes.c_int, vp, sz, vp],
            "tx_nccl_unique_id": [ctypes.c_char_p], "tx_nccl_init": [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, P(vp)],
            "tx_nccl_allreduce_sum": [vp, vp, sz, ctypes.c_int, vp], "tx_nccl_destroy": [vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        self._initialised = False

    # -- error handling ------------------------------------------------------
    def check(self, rc: int):
        if rc != 0:
            msg = (self.lib.tx_last_error() or b"").decode(errors="replace")
            raise DeviceError(rc, msg)

    def version(self) -> int:
        return self.lib.tx_version()

    def init(self, device: int = 0):
        if not self._initialised:
            self.check(self.lib.tx_init(device))
            self._initialised = True

    def device_info(self):
        a, b, c, m = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        self.check(self.lib.tx_device_info(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(m)))
        return {"sm_count": a.value, "cc": (b.value, c.value), "total_mem": m.value}

    # -- streams / events / graphs ---------------------------------------------
    def stream_create(self):
        s = ctypes.c_void_p()
        self.check(self.lib.tx_stream_create(ctypes.byref(s)))
        return s.value

    def stream_sync(self, s):
        self.check(self.lib.tx_stream_sync(s))

    def event_create(self):
        e = ctypes.c_void_p()
        self.check(self.lib.tx_event_create(ctypes.byref(e)))
        return e.value

    def event_record(self, e, s):
        self.check(self.lib.tx_event_record(e, s))

    def stream_wait_event(self, s, e):
        self.check(self.lib.tx_stream_wait_event(s, e))

    def event_sync(self, e):
        self.check(self.lib.tx_event_sync(e))

    def elapsed_ms(self, a, b) -> float:
        ms = ctypes.c_float()
        self.check(self.lib.tx_event_elapsed_ms(a, b, ctypes.byref(ms)))
        return ms.value

    def memcpy(self, dst, src, nbytes, kind, stream):
        self.check(self.lib.tx_memcpy_async(dst, src, nbytes, kind, stream))

    def memset(self, dst, value, nbytes, stream):
        self.check(self.lib.tx_memset_async(dst, value, nbytes, stream))

    def graph_begin(self, s):
        self.check(self.lib.tx_graph_begin(s))

    def graph_end(self, s):
        g = ctypes.c_void_p()
        self.check(self.lib.tx_graph_end(s, ctypes.byref(g)))
        return g.value

    def graph_launch(self, g, s):
        self.check(self.lib.tx_graph_launch(g, s))

    def graph_destroy(self, g):
        self.check(self.lib.tx_graph_destroy(g))

    def copy(self, src: TxTensor, dst: TxTensor, s):
        self.check(self.lib.tx_copy(ctypes.byref(src), ctypes.byref(dst), s))

    # -- kernels ------------------------------------------------------------
    def ew_compile(self, source: str, name: str):
        h = ctypes.c_void_p()
        self.check(self.lib.tx_ew_compile(source.encode(), name.encode(), ctypes.byref(h)))
        return h.value

    def kernel_compile(self, source: str, name: str, entry: str):
        h = ctypes.c_void_p()
        self.check(self.lib.tx_kernel_compile(source.encode(), name.encode(), entry.encode(), ctypes.byref(h)))
        return h.value

    def ew_check(self, source: str, name: str = "check") -> int:
        n = ctypes.c_size_t()
        self.check(self.lib.tx_ew_check(source.encode(), name.encode(), ctypes.byref(n)))
        return n.value

    def reduce_workspace(self, op, x: TxTensor, mask) -> int:
        n = ctypes.c_size_t()
        self.check(self.lib.tx_reduce_workspace(op, ctypes.byref(x), mask, ctypes.byref(n)))
        return n.value

    def gemm_workspace(self, a, b, c, mode=GEMM_AUTO) -> int:
        n = ctypes.c_size_t()
        self.check(self.lib.tx_gemm_workspace(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), mode,
                                              ctypes.byref(n)))
        return n.value

    def narrow_grad_workspace(self, dz, wt, h, dh, gw, db, mode=GEMM_AUTO) -> int:
        n = ctypes.c_size_t()
        self.check(self.lib.tx_narrow_grad_workspace(dz, wt, h, dh, gw, db, mode, ctypes.byref(n)))
        return n.value

    def gemm_path(self, a, b, c, mode=GEMM_AUTO) -> int:
        p = ctypes.c_int()
        self.check(self.lib.tx_gemm_path(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), mode, ctypes.byref(p)))
        return p.value

    # -- NCCL -----------------------------------------------------------------
    def nccl_unique_id(self) -> bytes:
        buf = ctypes.create_string_buffer(128)
        self.check(self.lib.tx_nccl_unique_id(buf))
        return buf.raw

    def nccl_init(self, nranks, rank, uid: bytes):
        c = ctypes.c_void_p()
        self.check(self.lib.tx_nccl_init(nranks, rank, uid, ctypes.byref(c)))
        return c.value


_lib = None
_lock = threading.Lock()


def library() -> Library:
    """The process-wide library handle (loaded, not yet device-initialised)."""
    global _lib
    with _lock:
        if _lib is None:
            _lib = Library()
        return _lib


def device_library(device: int | None = None) -> Library:
    """Library handle with the CUDA device initialised; raises without a GPU."""
    lib = library()
    if device is None:
        try:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:  # pragma: no cover
            device = 0
    lib.init(device)
    return lib
