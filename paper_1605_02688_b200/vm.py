"""The device VM: ``compile`` / ``CompiledFunction`` on B200.

Replaces the reference linker/VM (``runtime.py:174-553``), which walks a
Python thunk per node over NumPy arrays (~15 us of dispatch per node, SURVEY
F7) and copies every input in and every output out.  Here a call is:

  1. bind inputs (host arrays are copied H2D into plan-owned buffers; CUDA
     tensors are bound by pointer) and device-resident shared storage;
  2. look up / build a *step plan* for the (shapes, pointers, shared
     versions) signature: concrete shape inference with the reference's
     runtime checks, zero-copy views for DimShuffle, a liveness-planned arena
     (exact-size block reuse plus in-place reuse for elementwise kernels), and
     one launch closure per node calling the C ABI;
  3. replay the plan as one CUDA graph (captured on first use);
  4. copy the explicit outputs D2H.

Updates are written on the device: when every other reader of a shared
variable is scheduled before the update's producer (enforced with extra
scheduling edges, like the reference's destroy-before-read edges at
``runtime.py:305-317``) the producer writes straight into the shared storage;
otherwise the new value is committed by a copy after all reads.  There is no
host execution path.
"""
from __future__ import annotations

import threading
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np

from . import codegen, native
from .dtypes import ITEMSIZE, np_dtype
from .elemwise import Composite, Elemwise, EwProgram
from .shaping import IncSubtensor

# debugging aid (tests): TX_POISON=1 fills every arena / scratch buffer with NaN bytes
_POISON = bool(__import__("os").environ.get("TX_POISON"))
from .errors import (NotSupported, ShapeMismatch, TexprError, TypeMismatch,
                     UnderdeterminedOutputs)
from .graph import Constant, FunctionGraph, Variable, clone_outputs
from .op import UNKNOWN_SHAPE, is_host_op
from .rewrite import RewriteContext, run_preset
from .shared import SharedVariable, torch_dtype

INF = 1 << 60
ALIGN = 256
# cached step plans per function (distinct shape signatures; LRU beyond this)
MAX_PLANS = int(__import__("os").environ.get("TX_MAX_PLANS", "8"))


def _torch():
    import torch
    return torch


@dataclass(frozen=True)
class UpdatePair:
    shared: SharedVariable
    new_value: Variable


@dataclass
class Profile:
    call_count: int = 0
    total_time: float = 0.0
    _node_calls: dict = field(default_factory=dict)
    node_time: dict = field(default_factory=dict)
    node_bytes: dict = field(default_factory=dict)
    stage_times: dict = field(default_factory=dict)
    # whole-graph replays not yet folded into the per-node counts (a replay
    # runs every node once; folding lazily keeps the per-call cost O(1))
    _pending: int = 0
    _order: tuple = ()

    @property
    def node_calls(self):
        if self._pending:
            for nid in self._order:
                self._node_calls[nid] = self._node_calls.get(nid, 0) + self._pending
            self._pending = 0
        return self._node_calls

    def record_node(self, node_id, seconds, nbytes):
        self.node_calls[node_id] = self.node_calls.get(node_id, 0) + 1
        self.node_time[node_id] = self.node_time.get(node_id, 0.0) + seconds
        self.node_bytes[node_id] = self.node_bytes.get(node_id, 0) + nbytes

    def as_json(self, fn):
        return {"call_count": self.call_count, "total_time": self.total_time,
                "nodes": [{"id": n.id, "op": getattr(n.op, "display_name", n.op.name),
                           "calls": self.node_calls.get(n.id, 0), "time": self.node_time.get(n.id, 0.0),
                           "bytes": self.node_bytes.get(n.id, 0)} for n in fn.order],
                "stages": [{"stage": s, "time": t} for s, t in sorted(self.stage_times.items())]}

    def as_table(self, fn):
        rows = [f"calls: {self.call_count}   total: {self.total_time:.6f}s",
                f"{'op':<32}{'calls':>8}{'time (s)':>14}{'bytes':>14}"]
        for e in sorted(self.as_json(fn)["nodes"], key=lambda e: -e["time"]):
            rows.append(f"{e['op'][:31]:<32}{e['calls']:>8}{e['time']:>14.6f}{e['bytes']:>14}")
        return "\n".join(rows)


# ---------------------------------------------------------------------------
# storage & layouts

class Storage:
    __slots__ = ("kind", "nbytes", "offset", "ptr", "last_use", "alias", "name", "owner")

    def __init__(self, kind, nbytes=0, ptr=None, name=""):
        self.kind = kind          # arena | input | shared | const
        self.nbytes = nbytes
        self.offset = None
        self.ptr = ptr
        self.last_use = -1
        self.alias = None
        self.name = name
        self.owner = None         # torch tensor holding the memory, when plan-owned

    def root(self):
        s = self
        while s.alias is not None:
            s = s.alias
        return s


class Layout:
    __slots__ = ("storage", "offset", "shape", "strides", "dtype")

    def __init__(self, storage, offset, shape, strides, dtype):
        self.storage, self.offset = storage, offset
        self.shape, self.strides, self.dtype = tuple(shape), tuple(strides), dtype

    @property
    def numel(self):
        n = 1
        for s in self.shape:
            n *= s
        return n

    def contiguous(self) -> bool:
        exp = 1
        for s, st in zip(reversed(self.shape), reversed(self.strides)):
            if s != 1 and st != exp:
                return False
            exp *= s
        return True


def contiguous_strides(shape):
    st, acc = [], 1
    for s in reversed(shape):
        st.append(acc)
        acc *= s
    return tuple(reversed(st))


class ArenaAllocator:
    """Offsets for step-lifetime buffers: exact-size reuse, else first-fit."""

    def __init__(self):
        self.top = 0
        self.free: list[tuple[int, int]] = []

    def alloc(self, nbytes):
        n = max(ALIGN, (nbytes + ALIGN - 1) // ALIGN * ALIGN)
        best = None
        for i, (off, sz) in enumerate(self.free):
            if sz == n:
                best = i
                break
            if sz > n and (best is None or sz < self.free[best][1]):
                best = i
        if best is not None:
            off, sz = self.free.pop(best)
            if sz > n:
                self.free.append((off + n, sz - n))
            return off
        off = self.top
        self.top += n
        return off

    def release(self, off, nbytes):
        n = max(ALIGN, (nbytes + ALIGN - 1) // ALIGN * ALIGN)
        self.free.append((off, n))
        self.free.sort()
        merged = []
        for o, s in self.free:
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + s)
            else:
                merged.append((o, s))
        self.free = merged


# ---------------------------------------------------------------------------
# compile

def compile(inputs, outputs, updates=(), preset="fast_run", allow_gc=True, nan_guard=None, include=(),
            exclude=(), conv_impl="gemm", max_passes=8, *, cuda_graph=True, gemm_mode="auto",
            data_parallel=None, row_fusion=True) -> "CompiledFunction":
    """Build a callable computing ``outputs`` from ``inputs`` on the B200.

    Signature and semantics follow reference ``runtime.py:174-259``; extra
    keyword-only options: ``cuda_graph`` (capture/replay steps), ``gemm_mode``
    ("auto" tcgen05 TF32 where eligible | "simt" exact fp32 products) and
    ``data_parallel`` (a :class:`dp.DataParallel` group for synchronous
    gradient allreduce).
    """
    single = isinstance(outputs, Variable)
    outputs = [outputs] if single else list(outputs)
    inputs = list(inputs)
    ups = []
    for u in updates:
        pair = u if isinstance(u, UpdatePair) else UpdatePair(*u)
        if not isinstance(pair.shared, SharedVariable):
            raise TypeMismatch(f"update target {pair.shared!r} is not a shared variable")
        if pair.shared.type != pair.new_value.type:
            raise TypeMismatch(f"update for {pair.shared!r} has type {pair.new_value.type}, "
                               f"expected {pair.shared.type}")
        ups.append(pair)
    uvals = [p.new_value for p in ups]
    declared = {id(v) for v in inputs}
    found, seen, stack = [], set(), list(outputs + uvals)
    while stack:
        v = stack.pop()
        if v.id in seen or id(v) in declared:
            continue
        seen.add(v.id)
        if v.owner is not None:
            stack.extend(v.owner.inputs)
        elif isinstance(v, SharedVariable):
            found.append(v)
        elif not isinstance(v, Constant):
            raise UnderdeterminedOutputs(f"{v!r} is needed to compute the outputs but is neither an "
                                         "input nor a shared variable")
    found.sort(key=lambda v: v.id)
    full = inputs + found
    repl = {v: Variable(v.type, v.name) for v in full}
    cloned, _ = clone_outputs(outputs + uvals, repl, copy_free=True)
    fg = FunctionGraph([repl[v] for v in full], cloned)
    fg.protected_inputs = {repl[v] for v in found}
    ctx = RewriteContext(conv_impl=conv_impl, execution_bound=True, max_passes=max_passes,
                         data_parallel=data_parallel is not None)
    _, log = run_preset(fg, preset, include=include, exclude=exclude, ctx=ctx)
    return CompiledFunction(fg, len(outputs), [repl[v] for v in inputs], [(s, repl[s]) for s in found],
                            [(p.shared, cloned[len(outputs) + i]) for i, p in enumerate(ups)],
                            log, preset, single, allow_gc=allow_gc, cuda_graph=cuda_graph,
                            gemm_mode=gemm_mode, data_parallel=data_parallel, row_fusion=row_fusion,
                            nan_guard=nan_guard)


function = compile


class CompiledFunction:
    def __init__(self, fgraph, n_outputs, input_vars, shared_bindings, updates, rewrite_log, preset,
                 single_output=False, allow_gc=True, cuda_graph=True, gemm_mode="auto", data_parallel=None,
                 row_fusion=True, nan_guard=None):
        self.fgraph = fgraph
        self.n_outputs = n_outputs
        self.input_vars = list(input_vars)
        self.shared_bindings = list(shared_bindings)
        # update values are read from the rewritten graph's outputs (the
        # variables captured at clone time may have been replaced)
        self.updates = [(s, fgraph.outputs[n_outputs + i]) for i, (s, _) in enumerate(updates)]
        self.rewrite_log = rewrite_log
        self.preset = preset
        self.single_output = single_output
        self.allow_gc = allow_gc
        self.cuda_graph = cuda_graph
        self.gemm_mode = {"auto": native.GEMM_AUTO, "simt": native.GEMM_SIMT, "tc": native.GEMM_TC,
                          "3xtf32": native.GEMM_3XTF32}[gemm_mode]
        self.dp = data_parallel
        self.nan_guard = nan_guard
        self.row_fusion = row_fusion and nan_guard is None
        self.profile = Profile(stage_times=dict(rewrite_log.stage_times))
        self.has_lazy = False
        self._lock = threading.Lock()
        self._plans: OrderedDict = OrderedDict()   # shape key -> StepPlan, LRU, at most MAX_PLANS
        self._consts: dict[int, object] = {}
        self._stream = None
        self._comm_stream = None
        self._xfer = None
        self._pipes: OrderedDict = OrderedDict()
        self.pipelined = True
        self.profile_nodes = False
        self._direct, self.order = self._schedule()
        self.has_lazy = any(getattr(n.op, "lazy", False) for n in self.order)
        # integer division raises ZeroDivisionError from a device flag read after
        # the step: like the NaN guard, that must happen before any update lands
        self.has_int_div = any(codegen.has_int_div(getattr(n.op, "program", None)
                                                   or EwProgram.single(n.op.kernel, [x.type.dtype for x in n.inputs]))
                               for n in self.order if isinstance(n.op, (Elemwise, Composite)))
        if self.nan_guard is not None or self.has_lazy or self.has_int_div:
            self._direct = {}   # updates are committed only after the whole step (guard / lazy walk / flags) finished
        if self.has_lazy:
            self.row_fusion = False
            if self.dp is not None:
                raise NotSupported("lazy ops (ifelse / breakpoint) in a data-parallel step")
        self.profile._order = tuple(n.id for n in self.order)
        self._events = None
        self.thunks = {}
        # explicit scalar integer inputs that size a loop (scan n_steps): the
        # trip count is baked into the step plan, so their VALUES join its key
        from .scan import ScanOp
        in_pos = {v.id: i for i, v in enumerate(self.input_vars)}
        self._value_keyed = sorted({in_pos[n.inputs[0].id] for n in self.order
                                    if isinstance(n.op, ScanOp) and n.op.has_nsteps and n.inputs[0].id in in_pos})
        self.shard = None
        if self.dp is not None:
            from . import dp as _dp
            self.shard = _dp.propagate(self.order, self.dp.input_states(self.input_vars))
            for s, u in self.updates:
                if self.shard.state.get(u.id, _dp.REPLICATED) not in (_dp.REPLICATED, _dp.PARTIAL):
                    raise NotSupported(f"update of {s!r} depends on per-shard values without a reduction "
                                       "over the data-parallel axis")

    # -- scheduling --------------------------------------------------------
    def _schedule(self):
        """Toposort with update-in-place edges; returns (direct-write map, order)."""
        g = self.fgraph
        shared_var_of = {id(var): s for s, var in self.shared_bindings}
        outputs_set = {v.id for v in g.outputs[: self.n_outputs]}
        direct = {}
        extra = {}
        used_values = {}
        for s, u in self.updates:
            used_values[u.id] = used_values.get(u.id, 0) + 1
        for s, u in self.updates:
            var = next((v for sh, v in self.shared_bindings if sh is s), None)
            if var is None:
                continue  # a target nothing reads: written back after the step
            p = u.owner
            if p is None or used_values[u.id] > 1 or u.id in outputs_set:
                continue
            if getattr(p.op, "view_capable", False) or not hasattr(p.op, "lower"):
                continue
            # the shared value (or a view of it) must not be a returned output
            # nor another update's value (those read the old value after the step)
            if _aliases_output(g, var, self.n_outputs):
                continue
            if any(u2 is not u and (u2 is var or _is_view_of(u2, var)) for _, u2 in self.updates):
                continue
            readers = _readers_through_views(g, var)
            reads_self = p in readers
            if reads_self:
                # in place over the value it reads: fine for elementwise kernels and
                # for the SGD GEMM epilogue (each element read, then written, once)
                if not (isinstance(p.op, (Elemwise, Composite)) or getattr(p.op, "elementwise_in_place", False)):
                    continue
                if not getattr(p.op, "reads_before_writes", False) and \
                        any(x is not var and _is_view_of(x, var) for x in p.inputs):
                    continue
            others = [r for r in readers if r is not p]
            trial = dict(extra)
            trial[p] = set(trial.get(p, set())) | set(others)
            try:
                g.toposort(extra_deps=trial)
            except TexprError:
                continue
            extra = trial
            direct[u.id] = (s, var)
        order = g.toposort(extra_deps=extra or None)
        return direct, order

    # -- calling -------------------------------------------------------------
    def __call__(self, *values):
        with self._lock:
            return self._call(values, device_out=False)

    def call_device(self, *values, sync: bool = False):
        """Run with CUDA-tensor (or host) inputs; returns CUDA tensors that
        alias internal buffers until the next call.  No host sync unless asked."""
        with self._lock:
            return self._call(values, device_out=True, sync=sync)

    @property
    def output_vars(self):
        return self.fgraph.outputs[: self.n_outputs]

    def thunk_count(self, node_id):
        return self.profile.node_calls.get(node_id, 0)

    def _lib(self):
        lib = native.device_library()
        if self._stream is None:
            t = _torch()
            self._tstream = t.cuda.Stream()
            self._stream = self._tstream.cuda_stream
        return lib

    def _xfer_streams(self, lib):
        """(H2D, D2H) copy streams for chunk-pipelined host calls."""
        if self._xfer is None:
            self._xfer = (lib.stream_create(), lib.stream_create())
        return self._xfer

    def _call(self, values, device_out, sync=True):
        t0 = time.perf_counter()
        if len(values) != len(self.input_vars):
            raise TypeMismatch(f"function expects {len(self.input_vars)} inputs, got {len(values)}")
        lib = self._lib()
        t = _torch()
        binds = []
        for var, val in zip(self.input_vars, values):
            binds.append(_bind_input(var, val))
        shared_state = []
        for s, var in self.shared_bindings:
            dev = s.device_tensor()
            why = var.type.shape_matches(np_dtype(var.type.dtype), tuple(dev.shape))
            if why is not None:
                raise TypeMismatch(f"shared {s!r} holds a nonconforming value: {why}")
            shared_state.append((dev.data_ptr(), tuple(dev.shape), s.version))
        # plans are keyed on shapes (and the shared storages they bake in),
        # never on the caller's input pointers: a fresh device tensor per call
        # (a data loader) re-uses the plan through its input slots
        key = (tuple((b.shape, b.dev_ptr is not None) for b in binds), tuple(shared_state))
        if self._value_keyed:
            vals = {}
            for i in self._value_keyed:
                b = binds[i]
                src = b.tensor if b.tensor is not None else b.host
                vals[self.input_vars[i].id] = int(np.asarray(src.cpu() if hasattr(src, "cpu") else src).reshape(()))
            key = key + (tuple(sorted(vals.items())),)
            self._bound_values = vals
        if self.pipelined and not device_out and key not in self._plans:
            from . import stream as _stream
            pipe = self._pipes.get(key)
            if pipe is None and _stream.eligible(self, binds, device_out):
                try:
                    pipe = _stream.Pipeline(self, lib, binds)
                except _stream._NotChunkable:
                    pipe = False
                self._pipes[key] = pipe
                while len(self._pipes) > MAX_PLANS:
                    old = self._pipes.pop(next(iter(self._pipes)))
                    if old:
                        old.release()
            elif key in self._pipes:
                self._pipes.move_to_end(key)
            if pipe:
                outs = pipe.run(binds)
                self.profile._pending += 1
                self.profile.call_count += 1
                self.profile.total_time += time.perf_counter() - t0
                return outs[0] if self.single_output else outs
        plan = self._plans.get(key)
        if plan is not None and not plan.accepts(binds):
            # the caller moved to new device buffers: replace the pointer-bound
            # plan by one that copies device inputs into plan-owned slots
            self._evict(key)
            plan = StepPlan(self, lib, binds, key, slot_inputs=True)
            self._plans[key] = plan
        elif plan is None:
            plan = StepPlan(self, lib, binds, key)
            self._plans[key] = plan
            while len(self._plans) > MAX_PLANS:
                self._evict(next(iter(self._plans)))
        else:
            self._plans.move_to_end(key)
        stream = self._stream
        if self._events is None:
            self._events = (lib.event_create(), lib.event_create())
        cur = None
        if any(b.dev_ptr is not None for b in binds) or device_out:
            # order after the caller's stream (inputs produced there)
            cur = t.cuda.current_stream().cuda_stream
            lib.event_record(self._events[0], cur)
            lib.stream_wait_event(stream, self._events[0])
        plan.upload_inputs(binds, stream)
        if self.has_lazy:
            plan.run_lazy(stream, self.profile)
        elif self.profile_nodes:
            plan.run_profiled(stream, self.profile)
        else:
            plan.run(stream)
            self.profile._pending += 1
        if plan.guard_slots:
            plan.check_guard(stream)      # raises NanDetected before any update is committed
        if plan.commit_launches:
            if plan.flag is not None:
                plan.check_flags(stream)  # raises ZeroDivisionError before any update is committed
            plan.run_commits(stream)
        if device_out:
            outs = plan.device_outputs()
            lib.event_record(self._events[1], stream)
            lib.stream_wait_event(cur, self._events[1])
            if sync:
                lib.stream_sync(stream)
        else:
            outs = plan.download_outputs(stream)
        plan.check_flags()
        if plan.finish_updates():
            self._evict_stale()
        self.profile.call_count += 1
        self.profile.total_time += time.perf_counter() - t0
        return outs[0] if self.single_output else outs

    def _evict(self, key):
        """Drop one cached plan: wait for the function's stream (its arena is
        handed back to the caching allocator), free its captured graphs.
        Device outputs handed out earlier keep the arena alive themselves."""
        plan = self._plans.pop(key, None)
        if plan is not None:
            plan.release(self._stream)

    def _evict_stale(self):
        """Plans baked against a shared storage that has since been replaced."""
        live = {(s.device_tensor().data_ptr(), s.version) for s, _ in self.shared_bindings}
        for key in [k for k in self._plans if any((p, v) not in live for p, _, v in k[1])]:
            self._evict(key)

    # -- serialization (reference runtime.py:555-569) -------------------------
    def save(self) -> bytes:
        from .serialize import encode_function
        with self._lock:
            return encode_function(self)

    # -- copying (reference runtime.py:512-553) ------------------------------
    def copy(self, swap=None, carry_updates=True, share_intermediate_storage=False):
        swap = dict(swap or {})
        for old, new in swap.items():
            if old.type != new.type:
                raise TypeMismatch(f"swap for {old!r} has type {new.type}, expected {old.type}")
        twin = CompiledFunction.__new__(CompiledFunction)
        twin.__dict__.update(self.__dict__)
        twin.shared_bindings = [(swap.get(s, s), v) for s, v in self.shared_bindings]
        twin.updates = [(swap.get(s, s), v) for s, v in self.updates] if carry_updates else []
        twin._direct = {k: (swap.get(s, s), v) for k, (s, v) in self._direct.items()} if carry_updates else {}
        twin.profile = Profile(stage_times=dict(self.profile.stage_times), _order=self.profile._order)
        twin._lock = threading.Lock()
        if share_intermediate_storage and carry_updates:
            # one set of step plans (arenas, captured graphs) for both
            # functions, run under one lock on one stream so they never
            # overlap; plans are keyed on the shared storages they bake in,
            # so a twin with swapped shared variables gets its own entries
            twin._lock = self._lock
            return twin
        twin._events = None
        twin._plans = OrderedDict()
        twin._pipes = OrderedDict()
        twin._stream = None
        twin._comm_stream = None
        twin._xfer = None
        return twin

    @property
    def _keep(self):
        """The function's intermediate storage (reference ``runtime.py`` keeps
        per-node buffers there with ``allow_gc=False``): here the cached step
        plans, whose arenas hold every intermediate."""
        return self._plans


def save(fn: CompiledFunction) -> bytes:
    """``TXFN`` container bytes (reference ``runtime.py:563-564``)."""
    return fn.save()


def load(data: bytes, force_reoptimize: bool = False, **compile_options) -> CompiledFunction:
    """Rebuild a function from ``TXFN`` bytes (reference ``runtime.py:567-570``);
    files written by the reference load too."""
    from .serialize import decode_function
    return decode_function(data, force_reoptimize=force_reoptimize, **compile_options)


def native_dtype_code(dtype):
    from .dtypes import DTYPE_CODE
    return DTYPE_CODE[dtype]


def _is_view_of(x, base) -> bool:
    while x.owner is not None and getattr(x.owner.op, "view_capable", False):
        x = x.owner.inputs[0]
        if x is base:
            return True
    return False


def _readers_through_views(g, var):
    out, stack = set(), [var]
    while stack:
        v = stack.pop()
        for c in g.node_clients(v):
            if c.id not in g.nodes:
                continue
            if getattr(c.op, "view_capable", False):
                stack.extend(c.outputs)
            else:
                out.add(c)
    return out


def _aliases_output(g, var, n_outputs):
    outs = g.outputs[:n_outputs]
    return any(o is var or _is_view_of(o, var) for o in outs)


# ---------------------------------------------------------------------------
# input binding

class _Bind:
    __slots__ = ("shape", "dev_ptr", "host", "tensor", "dtype")


def _bind_input(var, val) -> _Bind:
    b = _Bind()
    b.dtype = var.type.dtype
    t = None
    try:
        import torch
        if isinstance(val, torch.Tensor):
            t = val
    except ImportError:  # pragma: no cover
        pass
    if t is not None:
        want = torch_dtype(var.type.dtype)
        if t.dtype != want:
            raise TypeMismatch(f"value for input {var!r} has dtype {t.dtype}, expected {var.type.dtype}")
        why = var.type.shape_matches(np_dtype(var.type.dtype), tuple(t.shape))
        if why is not None:
            raise TypeMismatch(f"value for input {var!r} rejected: {why}")
        b.shape = tuple(t.shape)
        if t.is_cuda:
            if not t.is_contiguous():
                t = t.contiguous()
            b.dev_ptr, b.host, b.tensor = t.data_ptr(), None, t
        else:
            b.dev_ptr, b.host, b.tensor = None, t.contiguous(), None
        return b
    try:
        arr = np.array(val, dtype=np_dtype(var.type.dtype), copy=None)
    except (ValueError, TypeError) as exc:
        raise TypeMismatch(f"bad value for input {var!r}: {exc}") from exc
    why = var.type.value_matches(arr)
    if why is not None:
        raise TypeMismatch(f"value for input {var!r} rejected: {why}")
    if var.type.dtype == "bool":
        arr = arr.astype(np.uint8)
    b.shape, b.dev_ptr, b.tensor = arr.shape, None, None
    b.host = np.ascontiguousarray(arr)
    return b


# ---------------------------------------------------------------------------
# the step plan

class StepPlan:
    def __init__(self, fn: CompiledFunction, lib, binds, key, shared_arena=None, out_binds=None,
                 slot_inputs=False):
        """``shared_arena``: a dict through which plans that never run
        concurrently (the unrolled steps of a loop, ``scan.py``) share one
        scratch arena allocation.  ``out_binds``: {var id: device pointer} --
        node outputs written straight into caller-owned memory (a loop's
        history slot) instead of the arena.  ``slot_inputs``: device inputs
        are copied into plan-owned slots every call (reference
        runtime.py:163-171 always copies) instead of being bound by pointer
        into the captured graph."""
        self.fn, self.lib = fn, lib
        self.subplans = []                   # step plans of loops lowered into this plan
        self.values = dict(getattr(fn, "_bound_values", None) or {})  # var id -> host value (loop trip counts)
        t = _torch()
        g = fn.fgraph
        self.lay: dict[int, Layout] = {}
        self.keep = []                       # torch tensors that must stay alive
        self.in_storage = []                 # (Storage, nbytes) for host-bound inputs
        self.dev_slots = []                  # (Storage, nbytes) for slot-copied device inputs
        self.slot_inputs = slot_inputs
        # device pointers baked into the plan (None: host input or slot)
        self.bound_ptrs = tuple(None if slot_inputs else b.dev_ptr for b in binds)
        self.ws: dict[int, tuple] = {}       # node id -> (Storage, nbytes)
        self.flag = None
        order = fn.order
        pos = {n.id: i for i, n in enumerate(order)}
        n_steps = len(order)

        # ---- bound storages: inputs, shared, constants
        for var, b in zip(fn.input_vars, binds):
            nb = int(np.prod(b.shape, dtype=np.int64)) * ITEMSIZE[var.type.dtype]
            if b.dev_ptr is not None and not slot_inputs:
                st = Storage("input", nb, ptr=b.dev_ptr, name=var.name or "")
            else:
                st = Storage("input", nb, name=var.name or "")
                buf = t.empty(max(nb, 1), dtype=t.uint8, device="cuda")
                self.keep.append(buf)
                st.ptr = buf.data_ptr()
                st.owner = buf
                (self.in_storage if b.dev_ptr is None else self.dev_slots).append((st, nb))
            self.lay[var.id] = Layout(st, 0, b.shape, contiguous_strides(b.shape), var.type.dtype)
        in_ids = {v.id for v in fn.input_vars}
        self.host_inputs = [(st, nb) for st, nb in self.in_storage]
        self.shared_storage = {}
        for s, var in fn.shared_bindings:
            if var.id in self.lay:  # also declared as an explicit input
                continue
            dev = s.device_tensor()
            self.keep.append(dev)   # baked into the graph: outlives a shape-changing set_value
            st = Storage("shared", dev.numel() * dev.element_size(), ptr=dev.data_ptr(), name=s.name or "")
            self.shared_storage[id(s)] = st
            self.lay[var.id] = Layout(st, 0, tuple(dev.shape), contiguous_strides(tuple(dev.shape)), var.type.dtype)
        for n in order:
            for x in n.inputs:
                if isinstance(x, Constant) and x.id not in self.lay:
                    self.lay[x.id] = self._const_layout(x)

        # ---- shapes and layouts, node by node
        direct = fn._direct
        partial_ids = set()
        partial_vars = []
        if fn.shard is not None:
            partial_ids = set(fn.shard.partial_vars)
        for n in order:
            ins = [self.lay[x.id] for x in n.inputs]
            shapes = [l.shape for l in ins]
            if getattr(n.op, "name", "") == "scan":
                n.op.check_runtime_shapes(n, shapes, self.values)
                outs = n.op.infer_shape(n, shapes, self.values)
            elif getattr(n.op, "uses_values", False):
                n.op.check_runtime_shapes(n, shapes)
                outs = n.op.infer_shape(n, shapes, self.values)
            else:
                n.op.check_runtime_shapes(n, shapes)
                outs = n.op.infer_shape(n, shapes)
            if getattr(n.op, "plan_value", False):
                self.values[n.outputs[0].id] = n.op.value(n, shapes)
            if is_host_op(n.op) and any(s is UNKNOWN_SHAPE or any(d is None for d in s) for s in outs):
                # a host plugin op without infer_shape: its output shapes come
                # from one host evaluation on zeros of the input shapes
                probe = n.op.perform([np.zeros(sh, dtype=np_dtype(x.type.dtype)) for sh, x in zip(shapes, n.inputs)])
                outs = [tuple(np.shape(r)) for r in probe]
            for o, s in zip(n.outputs, outs):
                if s is UNKNOWN_SHAPE or any(d is None for d in s):
                    raise NotSupported(f"cannot infer the runtime shape of {o!r} ({n.op.name})")
            alias = getattr(n.op, "output_aliases", None)
            if alias is not None:
                for o, k in zip(n.outputs, alias()):
                    self.lay[o.id] = ins[k]
                continue
            if getattr(n.op, "view_capable", False):
                base = ins[0]
                shape, strides, off = n.op.view_layout(n, [(base.shape, base.strides, base.offset)])
                self.lay[n.outputs[0].id] = Layout(base.storage, off, shape, strides, n.outputs[0].type.dtype)
                continue
            for o, s in zip(n.outputs, outs):
                s = tuple(int(d) for d in s)
                if o.id in partial_ids:
                    nb = int(np.prod(s, dtype=np.int64)) * ITEMSIZE[o.type.dtype]
                    st = Storage("bucket", nb, name="grad")
                    self.lay[o.id] = Layout(st, 0, s, contiguous_strides(s), o.type.dtype)
                    partial_vars.append((o, nb))
                    continue
                if out_binds and o.id in out_binds:
                    nb = int(np.prod(s, dtype=np.int64)) * ITEMSIZE[o.type.dtype]
                    st = Storage("bound", nb, ptr=out_binds[o.id], name="bound")
                    self.lay[o.id] = Layout(st, 0, s, contiguous_strides(s), o.type.dtype)
                    continue
                d = direct.get(o.id)
                if d is not None:
                    sh, var = d
                    slay = self.lay.get(var.id)
                    if slay is not None and slay.shape == s and slay.storage.kind == "shared":
                        self.lay[o.id] = Layout(slay.storage, 0, s, contiguous_strides(s), o.type.dtype)
                        continue
                nb = int(np.prod(s, dtype=np.int64)) * ITEMSIZE[o.type.dtype]
                st = Storage("arena", nb, name=getattr(n.op, "display_name", n.op.name))
                self.lay[o.id] = Layout(st, 0, s, contiguous_strides(s), o.type.dtype)
            wsb = self._workspace_bytes(n)
            if wsb:
                self.ws[n.id] = (Storage("arena", wsb, name="ws"), wsb)

        # ---- placement: a ZeroEmbed whose regions partition its output has
        # each value's producer write straight into its region (the producer
        # output becomes a strided view of the embed's storage): the LSTM BPTT
        # body assembles dz from four gate gradients with no copies at all
        self.placed = {}
        placed_st = set()
        if not fn.has_lazy and fn.nan_guard is None:
            from .shaping import ZeroEmbed, _slice_geometry
            out_ids = {v.id for v in g.outputs}
            for n in order:
                if not isinstance(n.op, ZeroEmbed):
                    continue
                lo = self.lay[n.outputs[0].id]
                if lo.storage.kind not in ("arena", "bound") or not lo.contiguous() or not n.op.partition(lo.shape):
                    continue
                ks = set()
                for k, (items, v) in enumerate(zip(n.op.regions, n.inputs[1:])):
                    p = v.owner
                    if (p is None or not isinstance(p.op, (Elemwise, Composite)) or v.id in out_ids
                            or v.id in partial_ids or len(g.node_clients(v)) != 1 or v in n.inputs[k + 2:]
                            or self.lay[v.id].storage.kind != "arena"):
                        continue
                    shape, strides, off = _slice_geometry(items, lo.shape, lo.strides, lo.offset)
                    if tuple(shape) != tuple(self.lay[v.id].shape):
                        continue
                    self.lay[v.id] = Layout(lo.storage, off, shape, strides, v.type.dtype)
                    ks.add(k)
                if ks:
                    self.placed[n.id] = ks
                    placed_st.add(id(lo.storage))

        # ---- tail: output snapshots, contiguous copies, update commits
        written = set()
        self.commits = []      # (src Layout, dst Layout)
        self.late_updates = [] # (shared, Layout) for shape-changing updates
        for s, u in fn.updates:
            var = next((v for sh, v in fn.shared_bindings if sh is s), None)
            ul = self.lay[u.id] if u.id in self.lay else self._const_layout(u)
            slay = self.lay.get(var.id) if var is not None else None
            if slay is not None and ul.storage is slay.storage and ul.offset == 0 \
                    and ul.strides == slay.strides and ul.shape == slay.shape:
                written.add(id(slay.storage))
                continue  # written in place (or identity update)
            if slay is not None and ul.shape == slay.shape:
                # (a value that is another view of the same storage -- A <- A.T
                # -- is snapshotted below before the commit overwrites it)
                self.commits.append((ul, slay))
                written.add(id(slay.storage))
            else:
                self.late_updates.append((s, ul))
        self.tail_copies = []  # (src, dst) executed before commits
        self.out_lays = []
        for v in g.outputs[: fn.n_outputs]:
            if isinstance(v, Constant) and v.id not in self.lay:
                self.out_lays.append(("const", v.value))
                continue
            lay = self.lay[v.id]
            if not lay.contiguous() or id(lay.storage) in written or lay.offset != 0:
                nb = lay.numel * ITEMSIZE[lay.dtype]
                dst = Layout(Storage("arena", nb, name="out"), 0, lay.shape, contiguous_strides(lay.shape), lay.dtype)
                self.tail_copies.append((lay, dst))
                lay = dst
            self.out_lays.append(("dev", lay))
        # a commit must not read storage that this call overwrites: snapshot it
        fixed = []
        for src, dst in self.commits:
            if id(src.storage) in written:
                nb = src.numel * ITEMSIZE[src.dtype]
                snap = Layout(Storage("arena", nb, name="snap"), 0, src.shape, contiguous_strides(src.shape), src.dtype)
                self.tail_copies.append((src, snap))
                src = snap
            fixed.append((src, dst))
        self.commits = fixed
        late = []
        for sh, ul in self.late_updates:
            if id(ul.storage) in written:  # e.g. B <- A while A is itself updated
                nb = ul.numel * ITEMSIZE[ul.dtype]
                snap = Layout(Storage("arena", nb, name="snap"), 0, ul.shape, contiguous_strides(ul.shape), ul.dtype)
                self.tail_copies.append((ul, snap))
                ul = snap
            late.append((sh, ul))
        self.late_updates = late

        # ---- liveness over storages
        def touch(lay_, step):
            r = lay_.storage
            r.last_use = max(r.last_use, step)

        for i, n in enumerate(order):
            for x in n.inputs:
                touch(self.lay[x.id], i)
        end = n_steps
        for src, dst in self.tail_copies:
            touch(src, end)
            touch(dst, INF)
        for src, dst in self.commits:
            touch(src, end + 1)
        for _, ul in self.late_updates:
            touch(ul, INF)
        for kind, lay in self.out_lays:
            if kind == "dev":
                touch(lay, INF)
        for v in g.outputs:
            if v.id in self.lay:
                touch(self.lay[v.id], INF)

        # ---- row fusion (softmax / cross-entropy regions), decided with shapes
        self.row_groups = []
        if fn.row_fusion:
            from . import rowfuse
            excl = {n.id for n in fn.shard.partial_nodes} if fn.shard is not None else set()
            self.row_groups = rowfuse.find_groups(self, order, g, excl)
            for grp in self.row_groups:
                # the group's kernel runs at its last member and the deferred
                # nodes right after it: everything they read or write (member
                # outputs included, even those only other members read) must
                # stay allocated until then
                for n in grp.members + grp.deferred:
                    for x in list(n.inputs) + list(n.outputs):
                        if x.id in self.lay:
                            touch(self.lay[x.id], grp.last_pos)

        # ---- arena allocation with in-place reuse for elementwise kernels
        deferred_ids = {n.id for grp in self.row_groups for n in grp.deferred}
        alloc = ArenaAllocator()
        # the zero-division flag is live for the whole step (cleared first,
        # read last): placed before any liveness-based reuse, never released
        if any(codegen.has_int_div(getattr(n.op, "program", None) or EwProgram.single(n.op.kernel, [x.type.dtype for x in n.inputs]))
               for n in order if isinstance(n.op, (Elemwise, Composite))):
            self.flag = Storage("arena", 4, name="flag")
            self.flag.offset = alloc.alloc(4)
        live_at: dict[int, list] = {}

        def assign(st, step=INF):
            if st.kind != "arena" or st.offset is not None or st.alias is not None:
                return
            st.offset = alloc.alloc(st.nbytes)
            if st.last_use < INF and step < INF:
                live_at.setdefault(max(st.last_use, step), []).append(st)

        for i, n in enumerate(order):
            if getattr(n.op, "view_capable", False):
                continue
            taken = set()
            is_inc = isinstance(n.op, IncSubtensor)
            inplace_ok = (isinstance(n.op, (Elemwise, Composite)) or is_inc) and fn.nan_guard is None \
                and not fn.has_lazy and not any(id(self.lay[o.id].storage) in placed_st for o in n.outputs)
            for o in n.outputs:
                ol = self.lay[o.id]
                st = ol.storage
                if st.kind != "arena" or st.offset is not None:
                    continue
                if inplace_ok:
                    # inc_subtensor updates its target in place when the target
                    # dies here (the BPTT gate-gradient assembly: a chain of
                    # region adds instead of a full copy per step)
                    cands = n.inputs[:1] if is_inc else n.inputs
                    if is_inc and self.lay[n.inputs[1].id].storage.root() is self.lay[n.inputs[0].id].storage.root():
                        cands = []
                    for x in cands:
                        xl = self.lay[x.id]
                        xs = xl.storage
                        # another operand reading the same storage through a
                        # different view (x * x.T) would see elements this
                        # kernel already overwrote: not in place
                        clash = any(self.lay[y.id].storage.root() is xs.root()
                                    and (self.lay[y.id].offset, self.lay[y.id].strides, self.lay[y.id].shape)
                                    != (xl.offset, xl.strides, xl.shape)
                                    for y in n.inputs if y is not x and y.id in self.lay)
                        # chains are allowed (an in-place value that is itself
                        # an alias): the buffer is the root's, and the value
                        # and the root must both die at this node
                        r = xs.root()
                        if (not clash and r.kind == "arena" and r.offset is not None and xs.kind == "arena"
                                and id(r) not in taken and xs.last_use == i and r.last_use == i
                                and xl.offset == 0 and xl.shape == ol.shape and xl.dtype == ol.dtype
                                and xl.contiguous() and xs.nbytes == st.nbytes and r.nbytes == st.nbytes):
                            st.alias = xs
                            taken.add(id(r))
                            r.last_use = max(r.last_use, st.last_use)
                            lst = live_at.get(i)
                            if lst and r in lst:
                                lst.remove(r)
                            if r.last_use < INF:
                                live_at.setdefault(r.last_use, []).append(r)
                            break
                if st.alias is None:
                    assign(st, i)
            w = self.ws.get(n.id)
            if w is not None:
                w[0].offset = alloc.alloc(w[1])
                # a node deferred past a row-fusion launch runs after its
                # schedule slot: its scratch must not be handed on from here
                if n.id not in deferred_ids:
                    alloc.release(w[0].offset, w[1])
            for st in live_at.pop(i, []):
                if fn.nan_guard is None and not fn.has_lazy:
                    # a guarded step keeps every value for its report; a lazy
                    # walk runs nodes out of schedule order
                    alloc.release(st.offset, st.nbytes)
        for src, dst in self.tail_copies:
            assign(dst.storage)
        # any arena storage not yet placed (e.g. unused outputs)
        for lay in list(self.lay.values()):
            assign(lay.storage.root())
        self.buckets = []  # (dtype, ptr, count, member vars)
        if partial_vars:
            from . import dp as _dp
            info = []
            for v, nb in sorted(partial_vars, key=lambda vn: pos[vn[0].owner.id]):
                uses = [pos[c.id] for c in g.node_clients(v)]
                info.append((v, nb, pos[v.owner.id], min(uses) if uses else None))
            for members in _dp.make_buckets(info, fn.dp.bucket_bytes):
                off, offs = 0, []
                for v in members:
                    offs.append(off)
                    off += self.lay[v.id].numel * ITEMSIZE[v.type.dtype]
                buf = t.zeros(max(off, ALIGN), dtype=t.uint8, device="cuda")
                self.keep.append(buf)
                for v, o in zip(members, offs):
                    st = self.lay[v.id].storage
                    st.ptr = buf.data_ptr() + o
                count = off // ITEMSIZE[members[0].type.dtype]
                self.buckets.append((members[0].type.dtype, buf.data_ptr(), count, members))
        self.arena_bytes = alloc.top
        need = max(alloc.top, ALIGN)
        if shared_arena is not None:
            cur = shared_arena.get("t")
            if cur is None or cur.numel() < need:
                cur = t.empty(need, dtype=t.uint8, device="cuda")
                shared_arena["t"] = cur
            self.arena = cur
        else:
            self.arena = t.empty(need, dtype=t.uint8, device="cuda")
        if _POISON:
            self.arena.fill_(0xFF)  # NaN / -1 everywhere: uninitialised reads show up in results
        base = self.arena.data_ptr()
        for lay in list(self.lay.values()) + [d for _, d in self.tail_copies]:
            r = lay.storage.root()
            if r.kind == "arena" and r.ptr is None:
                r.ptr = base + r.offset
        for st, _ in self.ws.values():
            st.ptr = base + st.offset
        if self.flag is not None:
            self.flag.ptr = base + self.flag.offset

        # ---- launch closures
        self.launches = []  # (node or None, fn)
        self._cur = None
        bucket_after, bucket_wait = {}, {}
        if self.buckets:
            comm = fn.dp.comm(lib)
            if fn._comm_stream is None:
                fn._comm_stream = lib.stream_create()
            for bi, (dt, ptr, count, members) in enumerate(self.buckets):
                last = max(pos[v.owner.id] for v in members)
                bucket_after.setdefault(last, []).append(bi)
                first_use = min((pos[c.id] for v in members for c in g.node_clients(v)), default=None)
                if first_use is not None:
                    bucket_wait.setdefault(first_use, []).append(bi)
            self._bucket_events = [(lib.event_create(), lib.event_create()) for _ in self.buckets]
        grouped = {n.id for grp in self.row_groups for n in grp.members}
        deferred = {n.id for grp in self.row_groups for n in grp.deferred}
        group_at = {grp.last_pos: grp for grp in self.row_groups}
        self.guard_slots = []
        self.row_sources = []        # generated row-fusion kernels (diagnostics)
        self.commit_launches = []
        self.lazy_copies = {}
        if fn.nan_guard is not None:
            n_slots = sum(len(n.inputs) + len(n.outputs) for n in order)
            self._guard_buf = t.zeros(max(n_slots, 1), dtype=t.int32, device="cuda")
            self.keep.append(self._guard_buf)
        for i, n in enumerate(order):
            for bi in bucket_wait.get(i, []):
                self._emit_bucket_wait(bi)
            if n.id in grouped:
                if i in group_at:
                    from . import rowfuse
                    self._cur = n
                    launch, _src = rowfuse.emit_group(self, group_at[i], g)
                    self.row_sources.append(_src)
                    self.add_launch(launch)
                    for d in group_at[i].deferred:
                        if not getattr(d.op, "view_capable", False):
                            self._cur = d
                            d.op.lower(d, self)
            elif n.id in deferred:
                continue
            elif not getattr(n.op, "view_capable", False):
                self._cur = n
                n.op.lower(n, self)
            if fn.nan_guard is not None:
                self._emit_guard(n)
            for bi in bucket_after.get(i, []):
                self._emit_allreduce(bi, comm)
        for bi in range(len(self.buckets)):
            self._emit_bucket_wait(bi)
        self._cur = None
        for src, dst in self.tail_copies:
            self._emit_copy(src, dst)
        for src, dst in self.commits:
            self._emit_copy(src, dst)
        if (fn.nan_guard is not None or fn.has_lazy or fn.has_int_div) and self.commits:
            # updates land only after the guard passed (reference runtime.py:415-421)
            n_commit = len(self.commits)
            self.commit_launches = [fn_ for _, fn_ in self.launches[-n_commit:]]
            del self.launches[-n_commit:]
        self.graph = None
        self.captured = False
        self._pinned_out = None
        self._dev_outs = None

    # -- helpers used by op.lower -------------------------------------------
    def _const_layout(self, c: Constant) -> Layout:
        cache = self.fn._consts
        ent = cache.get(c.id)
        if ent is None:
            t = _torch()
            arr = np.array(c.value, order="C", copy=True)
            if c.type.dtype == "bool":
                arr = arr.astype(np.uint8)
            dev = t.from_numpy(arr.copy()).to("cuda") if arr.size else t.empty(1, dtype=t.uint8, device="cuda")
            ent = dev
            cache[c.id] = ent
        st = Storage("const", c.value.nbytes, ptr=ent.data_ptr())
        return Layout(st, 0, c.value.shape, contiguous_strides(c.value.shape), c.type.dtype)

    def layout(self, var) -> Layout:
        return self.lay[var.id]

    def ptr_of(self, lay: Layout) -> int:
        """Device address of a layout's first element."""
        return lay.storage.root().ptr + lay.offset * ITEMSIZE[lay.dtype]

    def scratch(self, shape, dtype) -> Layout:
        """A contiguous step-lifetime device buffer outside the arena."""
        t = _torch()
        nb = int(np.prod(shape, dtype=np.int64)) * ITEMSIZE[dtype]
        buf = t.empty(max(nb, ALIGN), dtype=t.uint8, device="cuda")
        if _POISON:
            buf.fill_(0xFF)
        self.keep.append(buf)
        st = Storage("scratch", nb, ptr=buf.data_ptr(), name="scratch")
        return Layout(st, 0, tuple(shape), contiguous_strides(tuple(shape)), dtype)

    def tx(self, var_or_layout, shape=None, strides=None) -> native.TxTensor:
        lay = var_or_layout if isinstance(var_or_layout, Layout) else self.lay[var_or_layout.id]
        r = lay.storage.root()
        ptr = r.ptr + lay.offset * ITEMSIZE[lay.dtype]
        return native.make_tensor(ptr, lay.dtype, lay.shape if shape is None else shape,
                                  lay.strides if strides is None else strides)

    def workspace(self, node):
        w = self.ws.get(node.id)
        if w is None:
            return None, 0
        return w[0].ptr, w[1]

    def add_launch(self, fn):
        self.launches.append((self._cur, fn))

    def _workspace_bytes(self, n) -> int:
        from .linalg import Dot
        from .reduce import _Reduce
        if isinstance(n.op, _Reduce):
            x = self._tx_noptr(self.lay[n.inputs[0].id])
            mask = sum(1 << a for a in n.op.axes)
            if not mask:
                return 0
            return self.lib.reduce_workspace(n.op.tx_code, x, mask)
        if hasattr(n.op, "workspace_bytes"):
            return n.op.workspace_bytes(self, n)
        if isinstance(n.op, Dot) or hasattr(n.op, "gemm_operands"):
            a, b, c = self._dot_views(n, noptr=True)
            return self.lib.gemm_workspace(a, b, c, self.fn.gemm_mode)
        return 0

    def _tx_noptr(self, lay, shape=None, strides=None):
        return native.make_tensor(16, lay.dtype, lay.shape if shape is None else shape,
                                  lay.strides if strides is None else strides)

    def view_of(self, lay: Layout, shape, strides, offset) -> Layout:
        """A layout over ``lay``'s storage (used by ops that write into or read
        from sub-regions: inc_subtensor, join, scan histories)."""
        return Layout(lay.storage, offset, shape, strides, lay.dtype)

    # -- emitters ---------------------------------------------------------------
    def emit_fill_zero(self, lay: Layout):
        """Zero a contiguous layout (memset) -- ZeroEmbed without a partition."""
        lib = self.lib
        nb = lay.numel * ITEMSIZE[lay.dtype]
        if not lay.contiguous():
            raise NotSupported("zero fill of a strided layout")
        ptr = self.ptr_of(lay)

        def launch(stream):
            lib.memset(ptr, 0, nb, stream)
        self.add_launch(launch)

    def emit_copy_layouts(self, src: Layout, dst: Layout):
        """Strided device copy src -> dst (same shape), attributed to the
        node being lowered."""
        lib = self.lib
        s, d = self.tx(src), self.tx(dst)

        def launch(stream):
            lib.copy(s, d, stream)
        self.add_launch(launch)

    def emit_gemm(self, a: Layout, b: Layout, c: Layout, mode=None):
        """C = A . B over explicit (possibly strided) layouts, with its own
        step-lifetime workspace (convolution lowering)."""
        lib = self.lib
        A, B, C = self.tx(a), self.tx(b), self.tx(c)
        mode = self.fn.gemm_mode if mode is None else mode
        wsb = lib.gemm_workspace(A, B, C, mode)
        ws = None
        if wsb:
            t = _torch()
            buf = t.empty(wsb, dtype=t.uint8, device="cuda")
            self.keep.append(buf)
            ws = buf.data_ptr()
        epi = native.TxEpilogue()
        f = lib.lib.tx_gemm

        def launch(stream):
            lib.check(f(A, B, C, epi, mode, ws, wsb, stream))
        self.add_launch(launch)

    def emit_elementwise_tx(self, program: EwProgram, outs, ins):
        """Launch ``program`` over explicit tensor descriptors (views)."""
        lib = self.lib
        h = codegen.CACHE.get(lib, program)
        arr = (native.TxTensor * (len(outs) + len(ins)))(*outs, *ins)
        n_out, n_in = len(outs), len(ins)
        flag = self.flag.ptr if (self.flag is not None and codegen.has_int_div(program)) else None
        f = lib.lib.tx_ew_launch

        def launch(stream):
            lib.check(f(h, n_out, n_in, arr, flag, stream))
        self.add_launch(launch)

    def emit_elementwise(self, node, program: EwProgram):
        lib = self.lib
        h = codegen.CACHE.get(lib, program)
        ops = [self.tx(o) for o in node.outputs] + [self.tx(x) for x in node.inputs]
        arr = (native.TxTensor * len(ops))(*ops)
        n_out, n_in = len(node.outputs), len(node.inputs)
        flag = self.flag.ptr if (self.flag is not None and codegen.has_int_div(program)) else None
        f = lib.lib.tx_ew_launch

        def launch(stream):
            lib.check(f(h, n_out, n_in, arr, flag, stream))
        self.add_launch(launch)

    def emit_reduce(self, node, code, axes):
        from .reduce import TX_ARGMAX_ONEHOT
        lib = self.lib
        x = self.tx(node.inputs[0])
        y = self.tx(node.outputs[0])
        mask = 0
        for a in axes:
            mask |= 1 << a
        if code == TX_ARGMAX_ONEHOT and mask == 0:
            self.emit_elementwise(node, EwProgram([node.inputs[0].type.dtype], [(node.outputs[0].type.dtype, 1)],
                                                  [("second", [("in", 0), ("const", 0)], node.outputs[0].type.dtype)],
                                                  [("node", 0)]))
            return
        ws, wsb = self.workspace(node)
        f = lib.lib.tx_reduce

        def launch(stream):
            lib.check(f(code, x, mask, y, ws, wsb, stream))
        self.add_launch(launch)

    def _dot_views(self, node, noptr=False):
        a, b = node.inputs[:2]
        c = node.outputs[0]
        la, lb, lc = self.lay[a.id], self.lay[b.id], self.lay[c.id]
        mk = self._tx_noptr if noptr else self.tx
        # promote rank-1 operands to matrices
        if len(la.shape) == 2:
            A = mk(la)
        else:
            A = mk(la, (1, la.shape[0]), (0, la.strides[0]))
        if len(lb.shape) == 2:
            B = mk(lb)
        else:
            B = mk(lb, (lb.shape[0], 1), (lb.strides[0], 0))
        M = A.shape[0]
        N = B.shape[1]
        if len(lc.shape) == 2:
            C = mk(lc)
        elif len(lc.shape) == 1:
            C = mk(lc, (M, N), (lc.strides[0], 0) if len(la.shape) == 2 else (0, lc.strides[0]))
        else:
            C = mk(lc, (1, 1), (1, 1))
        return A, B, C

    def emit_dot(self, node, epilogue=None):
        lib = self.lib
        A, B, C = self._dot_views(node)
        ws, wsb = self.workspace(node)
        mode = self.fn.gemm_mode
        epi = epilogue if epilogue is not None else native.TxEpilogue()
        f = lib.lib.tx_gemm

        def launch(stream):
            lib.check(f(A, B, C, epi, mode, ws, wsb, stream))
        self.add_launch(launch)

    def _emit_guard(self, node):
        """Scan every float input and output of ``node`` (reference
        diagnostics.py:52-88: inputs first, then outputs)."""
        from .dtypes import is_float
        cfg = self.fn.nan_guard
        mode = cfg.mode()
        big = float(cfg.big_threshold) if cfg.big_threshold is not None else 0.0
        lib = self.lib
        f = lib.lib.tx_check_values
        base = self._guard_buf.data_ptr()
        for label, vs in (("input", node.inputs), ("output", node.outputs)):
            for k, v in enumerate(vs):
                if not is_float(v.type.dtype):
                    continue
                lay = self.lay[v.id] if v.id in self.lay else self._const_layout(v)
                if lay.numel == 0:
                    continue
                slot = len(self.guard_slots)
                self.guard_slots.append((node, f"{label} {k}", lay))
                tx = self.tx(lay)

                def launch(stream, tx=tx, slot=slot):
                    lib.check(f(tx, base, slot, mode, big, stream))
                self.launches.append((None, launch))

    def copy_launch(self, src: Layout, dst: Layout):
        lib = self.lib
        s, d = self.tx(src), self.tx(dst)

        def launch(stream):
            lib.copy(s, d, stream)
        return launch

    def host_copy(self, lay: Layout, stream) -> np.ndarray:
        """Synchronous device->host copy of one value of the running step."""
        self.lib.stream_sync(stream)
        arr = _torch_view(lay, self.tx(lay).data).cpu().numpy()
        return arr.astype(np.bool_) if lay.dtype == "bool" else arr

    def run_lazy(self, stream, profile):
        """Demand-driven walk (reference runtime.py:448-499): only the nodes
        the outputs need through the taken branches run; conditions are read
        on the host when an ifelse / breakpoint needs them."""
        from .control import Breakpoint, IfElse, read_scalar
        fn = self.fn
        g = fn.fgraph
        by_node = {}
        tail = []
        for node, launch in self.launches:
            if node is None:
                tail.append(launch)
            else:
                by_node.setdefault(node.id, []).append(launch)
        if self.flag is not None:
            self.lib.memset(self.flag.ptr, 0, 4, stream)
        if self.guard_slots:
            self.lib.memset(self._guard_buf.data_ptr(), 0, 4 * len(self.guard_slots), stream)
        avail = {v.id for v in g.inputs}
        for target in g.outputs:
            stack = [target]
            while stack:
                v = stack[-1]
                if v.id in avail or isinstance(v, Constant):
                    stack.pop()
                    continue
                node = v.owner
                if isinstance(node.op, IfElse):
                    cond = node.inputs[0]
                    if cond.id not in avail and not isinstance(cond, Constant):
                        stack.append(cond)
                        continue
                    pick = 1 if bool(read_scalar(self, cond, stream)) else 2
                    branch = node.inputs[pick]
                    if branch.id not in avail and not isinstance(branch, Constant):
                        stack.append(branch)
                        continue
                    self.lazy_copies[node.id][pick - 1](stream)
                else:
                    missing = [x for x in node.inputs if x.id not in avail and not isinstance(x, Constant)]
                    if missing:
                        stack.extend(missing)
                        continue
                    for launch in by_node.get(node.id, ()):
                        launch(stream)
                    if isinstance(node.op, Breakpoint):
                        cv = read_scalar(self, node.inputs[0], stream)
                        if bool(cv):
                            mon = [self.host_copy(self.lay[x.id] if x.id in self.lay else self._const_layout(x),
                                                  stream) for x in node.inputs[1:]]
                            node.op.fire(cv, mon)
                for o in node.outputs:
                    avail.add(o.id)
                profile.node_calls[node.id] = profile.node_calls.get(node.id, 0) + 1
                stack.pop()
        for launch in tail:
            launch(stream)

    def check_guard(self, stream):
        """Read the guard words of the step just run; raise ``NanDetected``
        for the first flagged tensor in execution order."""
        from .diagnostics import NanReport, check_name, summarize
        from .errors import NanDetected
        self.lib.stream_sync(stream)
        flags = self._guard_buf.cpu().numpy()
        hit = np.flatnonzero(flags[: len(self.guard_slots)])
        if hit.size == 0:
            return
        node, label, lay = self.guard_slots[int(hit[0])]
        arr = _torch_view(lay, self.tx(lay).data).cpu().numpy()
        trace = next((str(o.trace) for o in node.outputs if getattr(o, "trace", None) is not None), "")
        raise NanDetected(NanReport(node_id=node.id, op=getattr(node.op, "display_name", node.op.name),
                                    check=check_name(int(flags[hit[0]])), tensor=label, trace=trace,
                                    value_summary=summarize(arr)))

    def run_commits(self, stream):
        for fn_ in self.commit_launches:
            fn_(stream)

    def _emit_allreduce(self, bi, comm):
        lib, cs = self.lib, self.fn._comm_stream
        dt, ptr, count, _ = self.buckets[bi]
        ready, done = self._bucket_events[bi]
        code = native_dtype_code(dt)
        f = lib.lib.tx_nccl_allreduce_sum

        def launch(stream):
            lib.event_record(ready, stream)
            lib.stream_wait_event(cs, ready)
            lib.check(f(comm, ptr, count, code, cs))
            lib.event_record(done, cs)
        self.launches.append((None, launch))

    def _emit_bucket_wait(self, bi):
        if getattr(self, "_waited", None) is None:
            self._waited = set()
        if bi in self._waited:
            return
        self._waited.add(bi)
        lib = self.lib
        done = self._bucket_events[bi][1]

        def launch(stream):
            lib.stream_wait_event(stream, done)
        self.launches.append((None, launch))

    def emit_host_op(self, node):
        """A user plugin op with only a host ``perform`` (``op.is_host_op``):
        drain the stream, bring the inputs to the host, run ``perform``, write
        the results into the node's planned device buffers.  The step holding
        it runs eagerly (host code cannot be captured into a CUDA graph)."""
        lib, t = self.lib, _torch()
        ins = [(self.lay[x.id], self.ptr_of(self.lay[x.id])) for x in node.inputs]
        outs = [(self.lay[o.id], self.ptr_of(self.lay[o.id]), o) for o in node.outputs]
        self.host_ops = getattr(self, "host_ops", 0) + 1
        op = node.op

        def launch(stream):
            lib.stream_sync(stream)
            vals = []
            for lay, ptr in ins:
                v = _torch_view(lay, ptr).cpu().numpy()
                vals.append(v.astype(np.bool_) if lay.dtype == "bool" else v)
            res = op.perform(vals, None)
            keep = []
            for (lay, ptr, o), r in zip(outs, res):
                arr = np.array(r, dtype=np_dtype(lay.dtype), order="C")
                if arr.shape != lay.shape:
                    raise ShapeMismatch(f"{getattr(op, 'name', op)}: perform returned shape {arr.shape}, "
                                        f"planned {lay.shape}")
                if lay.dtype == "bool":
                    arr = arr.astype(np.uint8)
                keep.append(arr)
                if arr.nbytes:
                    lib.memcpy(ptr, arr.ctypes.data, arr.nbytes, 0, stream)
            lib.stream_sync(stream)
            del keep
        self.add_launch(launch)

    def _emit_copy(self, src: Layout, dst: Layout):
        lib = self.lib
        s, d = self.tx(src), self.tx(dst)

        def launch(stream):
            lib.copy(s, d, stream)
        self.launches.append((None, launch))

    # -- execution --------------------------------------------------------------
    def accepts(self, binds) -> bool:
        """Whether this plan can run these inputs (same shapes are given by
        the cache key): a pointer-bound plan only its own device buffers."""
        return self.slot_inputs or all(p is None or p == b.dev_ptr for p, b in zip(self.bound_ptrs, binds))

    def release(self, stream=None):
        """Free the captured graphs (this plan's and its loops') once the
        stream has drained; the arena goes back with the last reference."""
        if stream is not None:
            self.lib.stream_sync(stream)
        for sp in self.subplans:
            if hasattr(sp, "release"):
                sp.release()
        if self.graph is not None:
            self.lib.graph_destroy(self.graph)
            self.graph = None

    def upload_inputs(self, binds, stream):
        if self.dev_slots:
            devs = [b for b in binds if b.dev_ptr is not None]
            for (st, nb), b in zip(self.dev_slots, devs):
                self.lib.memcpy(st.ptr, b.dev_ptr, nb, 2, stream)
        hosts = [b for b in binds if b.dev_ptr is None]
        for (st, nb), b in zip(self.host_inputs, hosts):
            if nb == 0:
                continue
            if isinstance(b.host, np.ndarray):
                self.lib.memcpy(st.ptr, b.host.ctypes.data, nb, 0, stream)
            else:  # torch CPU tensor (pinned or not)
                self.lib.memcpy(st.ptr, b.host.data_ptr(), nb, 0, stream)
        self._host_refs = hosts  # keep sources alive until the stream is synced

    def _launch_all(self, stream):
        if self.flag is not None:
            self.lib.memset(self.flag.ptr, 0, 4, stream)
        if self.guard_slots:
            self.lib.memset(self._guard_buf.data_ptr(), 0, 4 * len(self.guard_slots), stream)
        for _, fn in self.launches:
            fn(stream)

    def run(self, stream):
        if not self.fn.cuda_graph or getattr(self, "host_ops", 0):
            self._launch_all(stream)
            return
        if self.graph is None:
            # first call runs eagerly (surfaces errors with a clean stack), then capture
            self._launch_all(stream)
            self.lib.graph_begin(stream)
            try:
                self._launch_all(stream)
            except BaseException:
                try:
                    self.lib.graph_end(stream)
                except Exception:
                    pass
                raise
            self.graph = self.lib.graph_end(stream)
            return
        self.lib.graph_launch(self.graph, stream)

    def run_profiled(self, stream, profile):
        lib = self.lib
        if self.flag is not None:
            lib.memset(self.flag.ptr, 0, 4, stream)
        if self.guard_slots:
            lib.memset(self._guard_buf.data_ptr(), 0, 4 * len(self.guard_slots), stream)
        ev = [lib.event_create() for _ in range(2)]
        for node, fn in self.launches:
            lib.event_record(ev[0], stream)
            fn(stream)
            lib.event_record(ev[1], stream)
            lib.stream_sync(stream)
            if node is not None:
                nb = sum(self.lay[o.id].numel * ITEMSIZE[o.type.dtype] for o in node.outputs)
                profile.record_node(node.id, lib.elapsed_ms(ev[0], ev[1]) * 1e-3, nb)
        for n in self.fn.order:
            if getattr(n.op, "view_capable", False):
                profile.record_node(n.id, 0.0, 0)

    def download_outputs(self, stream):
        """D2H of the explicit outputs into fresh pinned host blocks (torch's
        caching host allocator), returned as NumPy views — each call returns
        new arrays (reference runtime.py:412-414) without a host-side copy."""
        from .stream import HOST_POOL
        pins = []
        for kind, lay in self.out_lays:
            if kind != "dev":
                pins.append(None)
                continue
            nb = lay.numel * ITEMSIZE[lay.dtype]
            ptr, base = HOST_POOL.take(nb)
            if nb:
                self.lib.memcpy(ptr, self.tx(lay).data, nb, 1, stream)
            pins.append(base)
        self.lib.stream_sync(stream)
        self._host_refs = None
        outs = []
        for (kind, lay), pin in zip(self.out_lays, pins):
            if kind == "const":
                outs.append(np.array(lay, copy=True))
                continue
            nb = lay.numel * ITEMSIZE[lay.dtype]
            dt = np.uint8 if lay.dtype == "bool" else np_dtype(lay.dtype)
            arr = pin[:nb].view(dt).reshape(lay.shape)
            if lay.dtype == "bool":
                arr = arr.astype(np.bool_)
            outs.append(arr)
        return outs

    def device_outputs(self):
        if self._dev_outs is not None:
            return list(self._dev_outs)
        t = _torch()
        outs = []
        for kind, lay in self.out_lays:
            if kind == "const":
                outs.append(t.from_numpy(np.array(lay)).to("cuda"))
                continue
            outs.append(_torch_view(lay, self.tx(lay).data, owner=self))
        # the views alias plan-owned buffers at fixed addresses: build once;
        # each keeps the plan (its arena) alive after an eviction
        self._dev_outs = tuple(outs)
        return outs

    def check_flags(self, stream=None):
        stream = self.fn._stream if stream is None else stream
        for sp in self.subplans:
            sp.check_flags(stream)
        if self.flag is None:
            return
        t = _torch()
        self.lib.stream_sync(stream)
        v = t.empty(1, dtype=t.int32, pin_memory=True)
        self.lib.memcpy(v.data_ptr(), self.flag.ptr, 4, 1, stream)
        self.lib.stream_sync(stream)
        if int(v.item()):
            raise ZeroDivisionError("integer division by zero")

    def finish_updates(self) -> bool:
        """Commit shape-changing updates (fresh shared storage); True if any."""
        if not self.late_updates:
            return False
        t = _torch()
        self.lib.stream_sync(self.fn._stream)
        for s, ul in self.late_updates:
            view = _torch_view(ul, self.tx(ul).data)
            with s._lock:
                s._dev = view.clone()
                s.version += 1
        return True


def _torch_view(lay: Layout, ptr: int, owner=None):
    """A torch tensor aliasing device memory at ``ptr`` with ``lay``'s geometry."""
    t = _torch()
    dt = torch_dtype(lay.dtype)
    if lay.numel == 0:
        return t.empty(lay.shape, dtype=dt, device="cuda")
    span = 1 + sum((s - 1) * st for s, st in zip(lay.shape, lay.strides))
    return _wrap_device_pointer(ptr, span, dt, owner).as_strided(lay.shape, lay.strides)


def _wrap_device_pointer(ptr, numel, dtype, owner=None):
    """Wrap raw device memory (owned by a plan's arena / shared storage) as a
    torch tensor via __cuda_array_interface__ (no copy).  torch keeps the
    interface object alive with the storage, and it holds ``owner``."""
    t = _torch()
    typestr = {t.float32: "<f4", t.float64: "<f8", t.int32: "<i4", t.int64: "<i8", t.uint8: "|u1"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(numel),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    cai = _CAI()
    cai.owner = owner
    return t.as_tensor(cai, device="cuda")
