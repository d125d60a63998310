"""Device-resident shared variables (reference ``runtime.py:45-104``).

The value lives in one contiguous CUDA allocation for the variable's whole
life; compiled steps bind it by pointer (so it is baked into captured CUDA
graphs) and updates are written into it on the device.  ``get_value`` copies
device->host, ``set_value`` host->device in place when the shape is unchanged
(pointer stable, no re-capture) or into fresh storage otherwise (plans keyed
on the storage version re-capture).
"""
from __future__ import annotations

import threading

import numpy as np

from .dtypes import dtype_of_value, np_dtype
from .errors import TypeMismatch
from .graph import TensorType, Variable


def _torch():
    import torch
    return torch


TORCH_DTYPE = {}


def torch_dtype(dtype: str):
    if not TORCH_DTYPE:
        t = _torch()
        TORCH_DTYPE.update({"float32": t.float32, "float64": t.float64, "int32": t.int32,
                            "int64": t.int64, "bool": t.uint8})
    return TORCH_DTYPE[dtype]


class SharedVariable(Variable):
    def __init__(self, value, name=None, dtype=None, broadcastable=None):
        arr = np.asarray(value)
        if dtype is None:
            dtype = dtype_of_value(arr)
        arr = np.array(arr, dtype=np_dtype(dtype), copy=True)
        if broadcastable is None:
            broadcastable = (False,) * arr.ndim
        vtype = TensorType(dtype, broadcastable)
        why = vtype.value_matches(arr)
        if why is not None:
            raise TypeMismatch(f"initial value rejected: {why}")
        super().__init__(vtype, name)
        self._lock = threading.Lock()
        self._host = arr          # pending host value (before first device use)
        self._dev = None          # torch CUDA tensor once resident
        self.version = 0          # bumps when the storage pointer changes

    def __repr__(self):
        return f"<shared {self.name or f'shared{self.id}'}:{self.type}>"

    # -- device side -----------------------------------------------------
    def device_tensor(self):
        """The resident CUDA tensor (uploaded on first use)."""
        with self._lock:
            if self._dev is None:
                t = _torch()
                host = self._host
                if self.type.dtype == "bool":
                    host = host.astype(np.uint8)
                self._dev = t.from_numpy(np.array(host, order="C", copy=True)).to("cuda", non_blocking=False)
                self._host = None
                self.version += 1
            return self._dev

    @property
    def shape(self):
        with self._lock:
            return tuple(self._dev.shape) if self._dev is not None else self._host.shape

    # -- host API ---------------------------------------------------------
    def get_value(self, borrow: bool = False) -> np.ndarray:
        with self._lock:
            if self._dev is None:
                return self._host if borrow else self._host.copy()
            t = _torch()
            t.cuda.synchronize()
            out = self._dev.cpu().numpy()
            if self.type.dtype == "bool":
                out = out.astype(np.bool_)
            return out

    def set_value(self, value) -> None:
        try:
            arr = np.array(value, dtype=np_dtype(self.type.dtype), copy=True)
        except (ValueError, TypeError) as exc:
            raise TypeMismatch(f"cannot store value in {self!r}: {exc}") from exc
        why = self.type.value_matches(arr)
        if why is not None:
            raise TypeMismatch(f"value rejected for {self!r}: {why}")
        with self._lock:
            if self._dev is None:
                self._host = arr
                return
            t = _torch()
            src = t.from_numpy(arr.astype(np.uint8) if self.type.dtype == "bool" else arr)
            t.cuda.synchronize()
            if tuple(self._dev.shape) == arr.shape:
                self._dev.copy_(src)
            else:
                self._dev = src.to("cuda")
                self.version += 1


def shared(value, name=None, dtype=None, broadcastable=None) -> SharedVariable:
    return SharedVariable(value, name, dtype, broadcastable)


def set_shared(s: SharedVariable, value) -> None:
    s.set_value(value)


def get_shared(s: SharedVariable) -> np.ndarray:
    return s.get_value()
