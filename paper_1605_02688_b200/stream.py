"""Chunk-pipelined calls for host-resident elementwise graphs.

The reference copies every input into the runtime and every output out
(``runtime.py:163-171``, ``:412-417``) — for config 2 that is 4.3 GB in and
1.1 GB out per call, and on the device the kernel itself is < 1 ms, so a
host-array call is bound by PCIe.  When a compiled graph is purely
elementwise over one iteration space (every node an Elemwise/Composite, every
input and output of the same shape) the call is split along axis 0 into
chunks and run as a three-stage pipeline over a ring of device slots:

    H2D stream   : copy chunk i's inputs into slot i % R
    compute      : replay slot's captured step graph   (waits H2D of chunk i)
    D2H stream   : copy chunk i's outputs to the pinned result blocks

so the host→device copies, the kernel and the device→host copies of
different chunks overlap (PCIe is full duplex).  Every slot is an ordinary
:class:`vm.StepPlan` for the chunk shape, so the kernels and semantics are
exactly those of the unchunked call.
"""
from __future__ import annotations

import threading
import weakref

import numpy as np

from .dtypes import ITEMSIZE, np_dtype
from .elemwise import Composite, Elemwise
from .graph import Constant

MIN_BYTES = 64 << 20          # below this a single plan is faster
# input bytes per chunk: fewer, larger copies keep the copy engines busier (config 2
# end to end, pinned: 16 MB 55.7, 32 MB 58.5, 128 MB 64.9, 256 MB 65.2 GB/s)
CHUNK_IN_BYTES = int(__import__("os").environ.get("TX_CHUNK_MB", "128")) << 20
SLOTS = 3


def eligible(fn, binds, device_out) -> bool:
    if (device_out or fn.updates or fn.shared_bindings or fn.dp is not None or fn.profile_nodes
            or fn.nan_guard is not None):
        return False
    if not binds or any(b.dev_ptr is not None for b in binds):
        return False
    shape = binds[0].shape
    if len(shape) == 0 or shape[0] < 2 * SLOTS or any(b.shape != shape for b in binds):
        return False
    total = sum(int(np.prod(b.shape, dtype=np.int64)) * ITEMSIZE[b.dtype] for b in binds)
    if total < MIN_BYTES:
        return False
    for n in fn.order:
        if not isinstance(n.op, (Elemwise, Composite)):
            return False
        for x in n.inputs:
            if isinstance(x, Constant):
                cs = np.shape(x.value)
                if len(cs) == len(shape) and cs and cs[0] != 1:
                    return False
            elif x.type.ndim != len(shape):
                return False
    outs = fn.fgraph.outputs[: fn.n_outputs]
    return all(not isinstance(o, Constant) and o.type.ndim == len(shape) for o in outs)


class _Bind:
    __slots__ = ("shape", "dev_ptr", "host", "tensor", "dtype")

    def __init__(self, shape, dtype):
        self.shape, self.dtype = shape, dtype
        self.dev_ptr = self.host = self.tensor = None


class Pipeline:
    """Slot plans for one (full shape) signature."""

    def __init__(self, fn, lib, binds):
        from .vm import StepPlan
        t = _torch()
        self.fn, self.lib = fn, lib
        shape = binds[0].shape
        self.rows = shape[0]
        row_elems = int(np.prod(shape[1:], dtype=np.int64))
        in_row_bytes = sum(row_elems * ITEMSIZE[b.dtype] for b in binds)
        rows = max(1, CHUNK_IN_BYTES // max(in_row_bytes, 1))
        # keep every chunk boundary 256-byte aligned for all dtypes
        align = max(1, 256 // max(1, np.gcd(256, row_elems)))
        rows = max(align, rows // align * align)
        rows = min(rows, max(align, self.rows // SLOTS // align * align))
        self.chunk = rows
        self.row_elems = row_elems
        self.in_dtypes = [b.dtype for b in binds]
        self.slots = []
        for _ in range(SLOTS):
            cb = [_Bind((rows,) + tuple(shape[1:]), b.dtype) for b in binds]
            self.slots.append(StepPlan(fn, lib, cb, None))
        rem = self.rows % rows
        self.tail = None
        if rem:
            cb = [_Bind((rem,) + tuple(shape[1:]), b.dtype) for b in binds]
            self.tail = StepPlan(fn, lib, cb, None)
        self.out_specs = []
        for kind, lay in self.slots[0].out_lays:
            if kind != "dev" or lay.shape[1:] != tuple(shape[1:]) or lay.shape[0] != rows:
                raise _NotChunkable()
            self.out_specs.append(lay.dtype)
        # an output that is an input variable (compile([x, y], [x, x*y])) is
        # copied out of the slot's input buffer: the next H2D into that slot
        # must then also wait for the D2H, not just for the compute
        self.out_reads_input = any(lay.storage.root().kind == "input" for _, lay in self.slots[0].out_lays)
        # steady state keeps two result blocks per output in flight (the
        # caller's previous result + this call's); pin them now, not mid-stream
        for dt in self.out_specs:
            HOST_POOL.reserve(self.rows * self.row_elems * ITEMSIZE[dt], 2)
        self.ev = [[lib.event_create() for _ in range(3)] for _ in range(SLOTS + 1)]
        self.used = [False] * (SLOTS + 1)
        self.stage = None          # pinned staging per slot for pageable inputs (lazy)
        # capture every slot's step graph up front (first run is eager + capture)
        st = fn._stream
        for p in self.slots + ([self.tail] if self.tail else []):
            p.run(st)
        lib.stream_sync(st)
        del t

    def run(self, binds):
        fn, lib = self.fn, self.lib
        comp = fn._stream
        h2d, d2h = fn._xfer_streams(lib)
        shape = binds[0].shape
        outs = []
        for dt in self.out_specs:
            outs.append(HOST_POOL.take(self.rows * self.row_elems * ITEMSIZE[dt]))
        src = [(b.host.ctypes.data if isinstance(b.host, np.ndarray) else b.host.data_ptr()) for b in binds]
        in_rb = [self.row_elems * ITEMSIZE[d] for d in self.in_dtypes]
        # pageable inputs (NumPy arrays, unpinned tensors: the reference's own
        # call convention) are copied by host threads into pinned staging and
        # DMA'd from there -- the driver's own pageable path stages one copy at
        # a time and serialises with the host (13.8 GB/s for config 2)
        pageable = [isinstance(b.host, np.ndarray) or not b.host.is_pinned() for b in binds]
        staged = any(pageable)
        if staged:
            self._ensure_stage(in_rb)
            host_u8 = [(np.asarray(b.host) if isinstance(b.host, np.ndarray) else b.host.numpy()).reshape(-1)
                       .view(np.uint8) if pg else None for b, pg in zip(binds, pageable)]
        out_rb = [self.row_elems * ITEMSIZE[d] for d in self.out_specs]
        r0 = 0
        i = 0
        while r0 < self.rows:
            n = min(self.chunk, self.rows - r0)
            if n == self.chunk:
                si = i % SLOTS
                plan = self.slots[si]
            else:
                si = SLOTS
                plan = self.tail
            e_in, e_comp, e_out = self.ev[si]
            if self.used[si]:
                lib.stream_wait_event(h2d, e_comp)      # slot inputs no longer read
                if self.out_reads_input:
                    lib.stream_wait_event(h2d, e_out)   # ... not even by the D2H
            if staged:
                if self.used[si]:
                    lib.event_sync(e_in)                # the slot's staging was DMA'd already
                jobs = []
                for k, (u8, rb) in enumerate(zip(host_u8, in_rb)):
                    if u8 is not None:
                        jobs += _split_copy(self.stage_np[si][k], u8, r0 * rb, n * rb)
                for j in [_POOL.submit(np.copyto, d, s_) for d, s_ in jobs]:
                    j.result()
            for k, ((st, nb), s, rb) in enumerate(zip(plan.host_inputs, src, in_rb)):
                if nb:
                    if staged and pageable[k]:
                        lib.memcpy(st.ptr, self.stage[si][k].data_ptr(), n * rb, 0, h2d)
                    else:
                        lib.memcpy(st.ptr, s + r0 * rb, n * rb, 0, h2d)
            lib.event_record(e_in, h2d)
            lib.stream_wait_event(comp, e_in)
            if self.used[si]:
                lib.stream_wait_event(comp, e_out)      # slot outputs already copied out
            plan.run(comp)
            lib.event_record(e_comp, comp)
            lib.stream_wait_event(d2h, e_comp)
            for (kind, lay), (optr, _), rb in zip(plan.out_lays, outs, out_rb):
                lib.memcpy(optr + r0 * rb, plan.tx(lay).data, n * rb, 1, d2h)
            lib.event_record(e_out, d2h)
            self.used[si] = True
            r0 += n
            i += 1
        lib.stream_sync(d2h)
        lib.stream_sync(comp)
        for p in self.slots + ([self.tail] if self.tail else []):
            p.check_flags()
        res = []
        for dt, (_, base) in zip(self.out_specs, outs):
            npdt = np.uint8 if dt == "bool" else np_dtype(dt)
            nb = self.rows * self.row_elems * ITEMSIZE[dt]
            arr = base[:nb].view(npdt).reshape(shape)
            if dt == "bool":
                arr = arr.astype(np.bool_)
            res.append(arr)
        return res


    def _ensure_stage(self, in_rb):
        if self.stage is not None:
            return
        t = _torch()
        self.stage = [[t.empty(max(self.chunk * rb, 1), dtype=t.uint8, pin_memory=True) for rb in in_rb]
                      for _ in range(SLOTS + 1)]
        self.stage_np = [[b.numpy() for b in slot] for slot in self.stage]

    def release(self):
        self.lib.stream_sync(self.fn._stream)
        for p in self.slots + ([self.tail] if self.tail else []):
            p.release()


# host copy threads for pageable staging (np.copyto releases the GIL); up to 16:
# config 2 with pageable NumPy inputs 44.8 (8 threads) -> 49.2 GB/s (16)
_POOL = __import__("concurrent.futures", fromlist=["ThreadPoolExecutor"]).ThreadPoolExecutor(
    max_workers=int(__import__("os").environ.get("TX_STAGE_THREADS", 0)) or max(2, min(16, (__import__("os").cpu_count() or 2))),
    thread_name_prefix="tx-stage")
_PIECE = 2 << 20


def _split_copy(dst_u8, src_u8, off, nbytes):
    """(dst view, src view) pieces of about 2 MB for the copy threads."""
    out = []
    for a in range(0, nbytes, _PIECE):
        b = min(nbytes, a + _PIECE)
        out.append((dst_u8[a:b], src_u8[off + a: off + b]))
    return out


class _NotChunkable(Exception):
    pass


class HostBlockPool:
    """Pinned host blocks for returned outputs, recycled only when the NumPy
    arrays handed out over a block (and every view of them) are gone.

    Each call still returns new arrays (reference ``runtime.py:412-414``),
    but the D2H lands in page-locked memory that was registered once, not
    in a fresh cudaHostAlloc per call (0.4 s per GiB on the B200 hosts)."""

    def __init__(self):
        self._free: list = []        # (nbytes, tensor)
        self._lock = threading.Lock()

    def take(self, nbytes):
        t = _torch()
        nbytes = max(int(nbytes), 1)
        with self._lock:
            best = None
            for i, (sz, blk) in enumerate(self._free):
                if sz >= nbytes and sz <= 2 * nbytes and (best is None or sz < self._free[best][0]):
                    best = i
            if best is not None:
                sz, blk = self._free.pop(best)
            else:
                blk, sz = None, nbytes
        if blk is None:
            blk = t.empty(sz, dtype=t.uint8, pin_memory=True)
        # every array or view handed out keeps `hold` alive (it is the base
        # object at the end of any view chain); the block is recycled only
        # after `hold` is collected
        hold = _Hold(blk.data_ptr(), sz)
        base = np.asarray(hold)
        weakref.finalize(hold, self._give_back, sz, blk)
        return blk.data_ptr(), base

    def reserve(self, nbytes, count):
        t = _torch()
        nbytes = max(int(nbytes), 1)
        with self._lock:
            have = sum(1 for sz, _ in self._free if nbytes <= sz <= 2 * nbytes)
        for _ in range(count - have):
            blk = t.empty(nbytes, dtype=t.uint8, pin_memory=True)
            self._give_back(nbytes, blk)

    def _give_back(self, sz, blk):
        with self._lock:
            self._free.append((sz, blk))
            # bound the cache: keep the 8 most recent blocks
            if len(self._free) > 8:
                self._free.pop(0)


class _Hold:
    __slots__ = ("__array_interface__", "__weakref__")

    def __init__(self, ptr, nbytes):
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


HOST_POOL = HostBlockPool()


def _torch():
    import torch
    return torch
