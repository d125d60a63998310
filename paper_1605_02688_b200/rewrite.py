"""The staged rewrite engine and the canonicalisation rules.

API and staging follow reference ``rewrites/engine.py:26-325``: named rewrites
registered into fixed stages (canonicalize, stabilize, specialize,
abstract_select, inplace, scan); presets ``none`` / ``fast_compile`` /
``fast_run``; local rewrites iterate over a worklist to a fixed point under a
``max_passes`` cap, global ones see the whole graph; every application is
logged.  The rules in this module restate ``rewrites/algebra.py`` and
``rewrites/stability.py``.  Device-specific passes (convex fusion, GEMM
epilogue attachment) live in ``fusion.py`` and register into the same stages.
There are no ``inplace`` rules: buffer reuse is decided by the device memory
planner (``vm.py``), which subsumes destroy-map marking.
"""
from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .errors import CycleDetected, RewriteCycleDetected, TexprError
from .graph import Constant, FunctionGraph, ancestor_items, apply, fresh_id

STAGES = ("canonicalize", "stabilize", "specialize", "abstract_select", "inplace", "scan")
PRESETS = {"none": (), "fast_compile": ("canonicalize", "abstract_select"), "fast_run": STAGES}
DEFAULT_MAX_PASSES = 8


@dataclass
class RewriteContext:
    conv_impl: str = "gemm"
    execution_bound: bool = False
    max_passes: int = DEFAULT_MAX_PASSES
    data_parallel: bool = False   # gradients are partial sums: no update fusion into their GEMMs


@dataclass
class Rewrite:
    name: str
    stage: str
    kind: str  # "local" | "global"
    fn: object
    tags: tuple = ("default",)


REGISTRY: list[Rewrite] = []


def register_rewrite(name, stage, kind, tags=("default",)):
    if stage not in STAGES:
        raise ValueError(f"unknown stage {stage!r}")
    if kind not in ("local", "global"):
        raise ValueError(f"unknown rewrite kind {kind!r}")

    def deco(fn):
        REGISTRY.append(Rewrite(name, stage, kind, fn, tuple(tags)))
        return fn
    return deco


def find_rewrite(name):
    for r in REGISTRY:
        if r.name == name:
            return r
    raise KeyError(f"no rewrite named {name!r}")


@dataclass
class LogRecord:
    stage: str
    rewrite: str
    kind: str
    pass_index: int
    node_id: int | None = None
    replaced_op: str | None = None
    replacement_op: str | None = None
    created_node_ids: tuple = ()   # local rewrites: nodes the replacement imported (replay_log)


@dataclass
class RewriteLog:
    records: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    notes: list = field(default_factory=list)
    stage_times: dict = field(default_factory=dict)

    def add(self, rec):
        self.records.append(rec)

    def count(self, rewrite=None, stage=None) -> int:
        return sum(1 for r in self.records
                   if (rewrite is None or r.rewrite == rewrite) and (stage is None or r.stage == stage))

    def rewrite_names(self):
        return {r.rewrite for r in self.records}

    def summary(self):
        by_stage = {}
        for r in self.records:
            by_stage[r.stage] = by_stage.get(r.stage, 0) + 1
        return {"total": len(self.records), "by_stage": by_stage,
                "by_rewrite": {n: self.count(rewrite=n) for n in sorted(self.rewrite_names())},
                "stage_times": dict(self.stage_times), "warnings": list(self.warnings)}


def _dname(op):
    return getattr(op, "display_name", op.name)


def try_local(fgraph, rw, node, ctx):
    """Apply one local rewrite at one node: None (no match), False (rejected
    because it would create a cycle) or the list of replaced pairs."""
    pairs = rw.fn(fgraph, node, ctx)
    if not pairs:
        return None
    try:
        fgraph.replace_all(pairs, reason=rw.name)
    except CycleDetected:
        return False
    return pairs


class _Stage:
    def __init__(self, fgraph, stage, rewrites, ctx, log):
        self.g, self.stage, self.ctx, self.log = fgraph, stage, ctx, log
        self.locals = [r for r in rewrites if r.kind == "local"]
        self.globals = [r for r in rewrites if r.kind == "global"]
        self.pass_index = 0
        self.flips: dict = {}

    def run(self):
        for p in range(max(1, self.ctx.max_passes)):
            self.pass_index = p
            n = self._sweep_locals()
            for rw in self.globals:
                n += rw.fn(self.g, self.ctx, self._emitter(rw))
            if n == 0:
                return
        self.log.warnings.append(f"stage {self.stage} hit the {self.ctx.max_passes}-pass cap "
                                 "before reaching a fixed point")

    def _emitter(self, rw):
        def emit(node=None, replaced=None, replacement=None, created=None):
            self.log.add(LogRecord(self.stage, rw.name, "global", self.pass_index,
                                   None if node is None else node.id, replaced, replacement))
        emit.note = lambda text: self.log.notes.append(f"{rw.name}: {text}")
        return emit

    def _sweep_locals(self):
        if not self.locals:
            return 0
        order = self.g.toposort()
        work, queued = deque(order), {n.id for n in order}
        budget = max(1, self.ctx.max_passes) * max(len(order), 1) * 4
        applied = 0
        while work:
            if budget <= 0:
                self.log.warnings.append(f"stage {self.stage} exceeded its work budget; stopping early")
                break
            budget -= 1
            node = work.popleft()
            queued.discard(node.id)
            if node.id not in self.g.nodes:
                continue
            for rw in self.locals:
                res = try_local(self.g, rw, node, self.ctx)
                if res is None:
                    continue
                if res is False:
                    self.log.notes.append(f"{rw.name}: rejected at node {node.id}")
                    continue
                applied += 1
                old, new = res[0]
                src, dst = _dname(node.op), (_dname(new.owner.op) if new.owner else "<input>")
                self.log.add(LogRecord(self.stage, rw.name, "local", self.pass_index, node.id, src, dst,
                                       tuple(n.id for n in getattr(self.g, "imported", ()))))
                self._oscillation(rw, src, dst)
                for _, nv in res:
                    touched = list(self.g.node_clients(nv))
                    if nv.owner is not None and nv.owner.id in self.g.nodes:
                        touched.append(nv.owner)
                        touched += [x.owner for x in nv.owner.inputs
                                    if x.owner is not None and x.owner.id in self.g.nodes]
                    for t in touched:
                        if t.id not in queued:
                            work.append(t)
                            queued.add(t.id)
                break
        return applied

    def _oscillation(self, rw, src, dst):
        if src == dst:
            return
        c, _ = self.flips.get((src, dst), (0, rw.name))
        self.flips[(src, dst)] = (c + 1, rw.name)
        back = self.flips.get((dst, src))
        if back is not None and c + 1 >= 4 and back[0] >= 4:
            raise RewriteCycleDetected(f"rewrites {rw.name!r} and {back[1]!r} keep undoing each other "
                                       f"({src} <-> {dst})")


def _silent(*a, **k):
    return None


_silent.note = lambda text: None


def replay_log(fgraph: FunctionGraph, log: RewriteLog, var_mapping: dict, ctx=None) -> FunctionGraph:
    """Re-apply a recorded rewrite sequence to a copy of the graph it was
    recorded on (reference ``rewrites/engine.py:343-396``): ``var_mapping``
    maps the original's variables to the copy's (``clone_with_replacements``).
    Local records are re-matched at the mapped node and the nodes they create
    are mapped in import order; global rewrites run once per recorded
    invocation.  Rewrites are deterministic per site, so the copy ends
    op-isomorphic to the optimized original."""
    ctx = ctx or RewriteContext()
    node_map = {old.owner.id: new.owner for old, new in var_mapping.items()
                if old.owner is not None and new.owner is not None}
    last_global = None
    for rec in log.records:
        rw = find_rewrite(rec.rewrite)
        if rec.kind == "global":
            if (rec.rewrite, rec.pass_index, rec.stage) == last_global:
                continue
            last_global = (rec.rewrite, rec.pass_index, rec.stage)
            rw.fn(fgraph, ctx, _silent)
            continue
        last_global = None
        node = node_map.get(rec.node_id)
        if node is None or node.id not in fgraph.nodes:
            raise RewriteCycleDetected(f"replay lost track of node {rec.node_id} for {rec.rewrite}")
        res = try_local(fgraph, rw, node, ctx)
        if not res:
            raise RewriteCycleDetected(f"replay of {rec.rewrite} failed to re-match at node {rec.node_id}")
        created = list(getattr(fgraph, "imported", ()))
        if len(created) != len(rec.created_node_ids):
            raise RewriteCycleDetected(f"replay of {rec.rewrite} created {len(created)} nodes, "
                                       f"expected {len(rec.created_node_ids)}")
        for oid, n in zip(rec.created_node_ids, created):
            node_map[oid] = n
    return fgraph


def select_rewrites(preset, include=(), exclude=()):
    if preset not in PRESETS:
        raise ValueError(f"unknown preset {preset!r} (choose from {sorted(PRESETS)})")
    stages = PRESETS[preset]
    out = []
    for rw in REGISTRY:
        if rw.name in exclude:
            continue
        if rw.name in include or (rw.stage in stages and "default" in rw.tags):
            out.append(rw)
    return out


def run_preset(fgraph: FunctionGraph, preset="fast_run", include=(), exclude=(), ctx=None):
    from . import conv, fusion, scan  # noqa: F401  (register the device, loop and convolution passes)
    ctx = ctx or RewriteContext()
    log = RewriteLog()
    chosen = select_rewrites(preset, include, exclude)
    for stage in STAGES:
        rws = [r for r in chosen if r.stage == stage]
        if not rws:
            continue
        t0 = time.perf_counter()
        _Stage(fgraph, stage, rws, ctx, log).run()
        log.stage_times[stage] = log.stage_times.get(stage, 0.0) + time.perf_counter() - t0
        if stage == "abstract_select":
            _check_abstract(fgraph, ctx)
    return fgraph, log


def _check_abstract(fgraph, ctx):
    """Implementation selection with every convolution implementation
    excluded (``conv_impl="none"``) must not leave placeholders behind
    (reference ``rewrites/engine.py:328-340``)."""
    if ctx.conv_impl != "none":
        return
    from .conv import Conv2d
    left = [n for n in fgraph.nodes.values() if isinstance(n.op, Conv2d) and n.op.is_abstract]
    if left:
        from .errors import NoImplementationSelected
        raise NoImplementationSelected("implementation selection ran with every convolution implementation "
                                       f"excluded; {len(left)} placeholder node(s) remain")


def graph_signature(fgraph: FunctionGraph) -> tuple:
    """Structure of a graph up to variable identity (for comparisons)."""
    order = fgraph.toposort()
    ref = {v.id: ("in", i) for i, v in enumerate(fgraph.inputs)}

    def r(x):
        if x.id in ref:
            return ref[x.id]
        if isinstance(x, Constant):
            return ("const", x.type.dtype, x.value.shape, x.value.tobytes())
        return ("dangling", x.id)

    entries = []
    for i, n in enumerate(order):
        entries.append((n.op.name, n.op.attrs_key(), tuple(r(x) for x in n.inputs)))
        for j, o in enumerate(n.outputs):
            ref[o.id] = ("node", i, j)
    return tuple(entries), tuple(r(v) for v in fgraph.outputs)


# ---------------------------------------------------------------------------
# canonicalize (reference rewrites/algebra.py)

COMMUTATIVE = ("add", "mul", "maximum")


def _kernel(node):
    from .elemwise import Elemwise
    return node.op.kernel if isinstance(node.op, Elemwise) else None


@register_rewrite("merge_duplicates", "canonicalize", "global")
def merge_duplicates(fgraph, ctx, emit) -> int:
    """CSE: unify equal constants, then nodes with equal (op, inputs)."""
    total = 0
    while True:
        changed = 0
        canon: dict = {}
        seen_ids = set()
        for n in fgraph.toposort():
            for x in n.inputs:
                if not isinstance(x, Constant) or x.id in seen_ids or x not in fgraph.clients:
                    continue
                c = canon.setdefault((x.type, x.signature()), x)
                if c is not x:
                    seen_ids.add(x.id)
                    fgraph.replace(x, c, "merge_duplicates")
                    changed += 1
        first: dict = {}
        for n in fgraph.toposort():
            if n.id not in fgraph.nodes:
                continue
            key = (n.op, tuple(x.id for x in n.inputs))
            c = first.get(key)
            if c is None:
                first[key] = n
                continue
            fgraph.replace_all(list(zip(n.outputs, c.outputs)), "merge_duplicates")
            emit(node=n, replaced=_dname(n.op), replacement=_dname(c.op))
            changed += 1
        total += changed
        if not changed:
            return total


def fold_node(node):
    """Compile-time evaluation of a node whose inputs are all small constants."""
    if not node.op.foldable or not node.inputs or not all(isinstance(x, Constant) for x in node.inputs):
        return None
    try:
        vals = node.op.fold([x.value for x in node.inputs])
    except (TexprError, ZeroDivisionError, FloatingPointError, ValueError):
        return None
    if vals is None:
        return None
    return [(o, Constant(np.asarray(v), dtype=o.type.dtype, broadcastable=o.type.broadcastable))
            for o, v in zip(node.outputs, vals)]


@register_rewrite("constant_fold", "canonicalize", "local")
def constant_fold(fgraph, node, ctx):
    return fold_node(node)


def _all_eq(c, value):
    return bool(np.all(c.value == value))


@register_rewrite("add_zero", "canonicalize", "local")
def add_zero(fgraph, node, ctx):
    if _kernel(node) != "add":
        return None
    out = node.outputs[0]
    for i in (0, 1):
        z, keep = node.inputs[i], node.inputs[1 - i]
        if isinstance(z, Constant) and _all_eq(z, 0) and keep.type == out.type:
            return [(out, keep)]
    return None


def _is_zeros(v) -> bool:
    """A zero tensor: a zero constant or ``zeros_like`` (second(x, 0))."""
    if isinstance(v, Constant):
        return _all_eq(v, 0)
    n = v.owner
    return (n is not None and getattr(n.op, "kernel", None) == "second" and isinstance(n.inputs[1], Constant)
            and _all_eq(n.inputs[1], 0))


@register_rewrite("add_into_zero_inc", "canonicalize", "local")
def add_into_zero_inc(fgraph, node, ctx):
    """add(X, inc_subtensor(zeros, v, region)) -> inc_subtensor(X, v, region)
    (B200-specific, not a reference rewrite).  ``grad`` of k slices of one
    tensor -- the LSTM's four gates -- gives a sum of k region-embedded
    gradients, each a full zero tensor plus a region; as a chain of
    inc_subtensors the planner updates one buffer in place (k region adds)
    instead of materialising k full tensors and summing them.  Values are
    unchanged (X + 0 = X off the region) up to the sign of a -0.0 in X."""
    from .shaping import IncSubtensor, inc_subtensor
    if _kernel(node) != "add":
        return None
    out = node.outputs[0]
    for i in (0, 1):
        inc, other = node.inputs[i], node.inputs[1 - i]
        n = inc.owner
        if n is None or not isinstance(n.op, IncSubtensor) or not _is_zeros(n.inputs[0]):
            continue
        if other.type != out.type or inc.type != out.type or len(fgraph.node_clients(inc)) != 1:
            continue
        return [(out, inc_subtensor(other, n.inputs[1], n.op.items))]
    return None


@register_rewrite("mul_one", "canonicalize", "local")
def mul_one(fgraph, node, ctx):
    if _kernel(node) != "mul":
        return None
    out = node.outputs[0]
    for i in (0, 1):
        one, keep = node.inputs[i], node.inputs[1 - i]
        if isinstance(one, Constant) and _all_eq(one, 1) and keep.type == out.type:
            return [(out, keep)]
    return None


@register_rewrite("mul_self_to_sqr", "canonicalize", "local")
def mul_self_to_sqr(fgraph, node, ctx):
    from .elemwise import make
    if _kernel(node) != "mul" or node.inputs[0] is not node.inputs[1]:
        return None
    return [(node.outputs[0], make("sqr", [node.inputs[0]]))]


@register_rewrite("neg_neg", "canonicalize", "local")
def neg_neg(fgraph, node, ctx):
    if _kernel(node) != "neg":
        return None
    inner = node.inputs[0].owner
    if inner is None or _kernel(inner) != "neg":
        return None
    x = inner.inputs[0]
    return [(node.outputs[0], x)] if x.type == node.outputs[0].type else None


def _div_cancel_match(node):
    if _kernel(node) != "div":
        return None
    num, den = node.inputs
    m = num.owner
    if m is None or _kernel(m) != "mul":
        return None
    for i in (0, 1):
        y, x = m.inputs[i], m.inputs[1 - i]
        same = y is den or (isinstance(y, Constant) and isinstance(den, Constant)
                            and y.signature() == den.signature())
        if same and x.type == node.outputs[0].type:
            return x, y
    return None


@register_rewrite("div_cancel", "canonicalize", "local")
def div_cancel(fgraph, node, ctx):
    m = _div_cancel_match(node)
    if m is None or not (isinstance(m[1], Constant) and bool(np.all(m[1].value != 0))):
        return None
    return [(node.outputs[0], m[0])]


@register_rewrite("div_cancel_unsafe", "canonicalize", "local", tags=("unsafe",))
def div_cancel_unsafe(fgraph, node, ctx):
    m = _div_cancel_match(node)
    return None if m is None else [(node.outputs[0], m[0])]


@register_rewrite("commutative_sort", "canonicalize", "local")
def commutative_sort(fgraph, node, ctx):
    if _kernel(node) not in COMMUTATIVE:
        return None
    a, b = node.inputs
    ca, cb = isinstance(a, Constant), isinstance(b, Constant)
    if (ca and not cb) or (ca == cb and a.id > b.id):
        return [(node.outputs[0], apply(node.op, [b, a])[0])]
    return None


@register_rewrite("log1p_stabilize", "stabilize", "local")
def log1p_stabilize(fgraph, node, ctx):
    from .elemwise import make
    if _kernel(node) != "log":
        return None
    add = node.inputs[0].owner
    if add is None or _kernel(add) != "add":
        return None
    out = node.outputs[0]
    for i in (0, 1):
        one, x = add.inputs[i], add.inputs[1 - i]
        if isinstance(one, Constant) and _all_eq(one, 1):
            r = make("log1p", [x])
            if r.type == out.type:
                return [(out, r)]
    return None


@register_rewrite("pow_specialize", "specialize", "local")
def pow_specialize(fgraph, node, ctx):
    from .elemwise import make
    if _kernel(node) != "pow":
        return None
    x, e = node.inputs
    if not (isinstance(e, Constant) and e.value.ndim == 0):
        return None
    v, out = float(e.value), node.outputs[0]
    if v == 1.0:
        r = x
    elif v == 2.0:
        r = make("sqr", [x])
    elif v == 0.5:
        r = make("sqrt", [x])
    else:
        return None
    return [(out, r)] if r.type == out.type else None


def created_since(watermark, roots):
    vs, ns = ancestor_items(roots)
    return [v for v in vs if v.id > watermark], [n for n in ns if n.id > watermark]


__all__ = ["STAGES", "PRESETS", "RewriteContext", "RewriteLog", "register_rewrite", "run_preset",
           "find_rewrite", "graph_signature", "REGISTRY", "fresh_id"]
