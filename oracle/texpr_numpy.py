"""NumPy restatement of texpr's host kernels and interpreter (test oracle).

Every function cites the reference line it restates.  The graph walker works
on any graph built with ``paper_1605_02688_b200`` (duck-typed on op names and
attributes), exactly like the reference's ``interp.eval_graph`` walks its own
graphs; ``eval_composite_chunked`` restates the reference's fused-Composite
execution so the CPU baseline times the reference algorithm.
"""
from __future__ import annotations

import heapq

import numpy as np

_ERR = {"divide": "ignore", "invalid": "ignore", "over": "ignore", "under": "ignore"}  # ops/elemwise.py:36
CHUNK = 1 << 15  # ops/elemwise.py:449


def stable_sigmoid(x):
    """ops/elemwise.py:44-46"""
    z = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + z), z / (1.0 + z))


def div(a, b, out=None):
    """ops/elemwise.py:49-55 — integer floor division raising on zero."""
    if a.dtype.kind in "iub" or b.dtype.kind in "iub":
        if np.issubdtype(np.result_type(a, b), np.integer):
            if np.any(b == 0):
                raise ZeroDivisionError("integer division by zero")
            return np.floor_divide(a, b, out=out)
    return np.true_divide(a, b, out=out)


def second(a, b):
    """ops/elemwise.py:76-81"""
    out = np.empty(np.broadcast_shapes(a.shape, b.shape), dtype=np.result_type(a, b))
    np.copyto(out, b)
    return out


# ops/elemwise.py:91-113 (name -> (fn, accepts out=, bool result))
KERNELS = {
    "add": (np.add, True, False), "sub": (np.subtract, True, False), "mul": (np.multiply, True, False),
    "div": (div, True, False), "neg": (np.negative, True, False), "exp": (np.exp, True, False),
    "log": (np.log, True, False), "log1p": (np.log1p, True, False), "pow": (np.power, True, False),
    "sqr": (np.square, True, False), "sqrt": (np.sqrt, True, False),
    "sigmoid": (stable_sigmoid, False, False), "tanh": (np.tanh, True, False),
    "maximum": (np.maximum, True, False), "switch": (lambda c, a, b: np.where(c, a, b), False, False),
    "second": (second, False, False),
    "lt": (np.less, True, True), "gt": (np.greater, True, True), "le": (np.less_equal, True, True),
    "ge": (np.greater_equal, True, True), "eq": (np.equal, True, True), "neq": (np.not_equal, True, True),
    "isnan": (np.isnan, True, True),
}


def elemwise(kernel, args, out=None):
    """Elemwise.perform (ops/elemwise.py:314-326)."""
    fn, ufunc, bool_out = KERNELS[kernel]
    with np.errstate(**_ERR):
        if ufunc:
            r = fn(*args, out=out)
        else:
            r = fn(*args)
            if out is not None:
                np.copyto(out, r)
                r = out
    if bool_out and r.dtype != np.bool_:
        r = r.astype(np.bool_)
    return r


def reduce_sum(x, axes):
    """Sum.perform (ops/reductions.py:91-101)."""
    return x.copy() if not axes else np.asarray(np.add.reduce(x, axis=tuple(axes)))


def reduce_max(x, axes):
    """Max.perform (ops/reductions.py:119-129)."""
    return x.copy() if not axes else np.asarray(np.maximum.reduce(x, axis=tuple(axes)))


def _moved(x, axes):
    others = [i for i in range(x.ndim) if i not in axes]
    perm = others + list(axes)
    moved = x.transpose(perm)
    return moved, perm, moved.shape[: len(others)]


def argmax_onehot(x, axes):
    """ArgmaxOnehot.perform (ops/reductions.py:166-179): first max, NaN wins."""
    if not axes:
        return np.ones_like(x)
    moved, perm, lead = _moved(x, axes)
    flat = moved.reshape(lead + (-1,))
    onehot = np.zeros_like(flat)
    idx = np.argmax(flat, axis=-1)
    np.put_along_axis(onehot, np.expand_dims(idx, -1), 1, axis=-1)
    return onehot.reshape(moved.shape).transpose(np.argsort(perm))


def argmax_index(x, axes):
    """Index form of the same np.argmax over the moved/reshaped view
    (ops/reductions.py:170-176), int64."""
    moved, perm, lead = _moved(x, axes)
    return np.asarray(np.argmax(moved.reshape(lead + (-1,)), axis=-1)).astype(np.int64)


def dot(a, b):
    """Dot.perform (ops/linalg.py:42-62): np.dot -> BLAS sgemm/sgemv/sdot."""
    return np.asarray(np.dot(a, b))


def dimshuffle(x, pattern):
    """DimShuffle.perform (ops/shaping.py:59-67)."""
    kept = [p for p in pattern if p != "x"]
    dropped = [i for i in range(x.ndim) if i not in kept]
    y = x.transpose(kept + dropped)
    idx = tuple([slice(None) if p != "x" else None for p in pattern] + [0] * len(dropped))
    return y[idx]


# ---------------------------------------------------------------- composites

def _program_eval(prog, env_in, targets=None):
    vals = []

    def get(ref):
        kind, i = ref
        if kind == "in":
            return env_in[i]
        if kind == "const":
            d, v = prog.consts[i]
            return np.asarray(v, dtype=np.dtype(d))
        return vals[i]

    for j, (k, refs, dt) in enumerate(prog.nodes):
        out = None if targets is None else targets.get(j)
        vals.append(elemwise(k, [get(r) for r in refs], out=out))
    return [get(r) for r in prog.outputs]


def eval_composite_plain(prog, inputs):
    """CompositeElemwise._perform_plain (ops/elemwise.py:546-556)."""
    return [np.asarray(v) for v in _program_eval(prog, inputs)]


def eval_composite_chunked(prog, inputs):
    """CompositeElemwise._perform_chunked (ops/elemwise.py:558-597): 32768-
    element chunks, one scratch buffer per inner node."""
    shape, size = inputs[0].shape, inputs[0].size
    flats = [a.reshape(-1) for a in inputs]
    outs = [np.empty(shape, dtype=np.dtype(d)) for d in prog.out_dtypes]
    out_flat = [o.reshape(-1) for o in outs]
    out_of = {}
    for oi, (kind, i) in enumerate(prog.outputs):
        if kind == "node":
            out_of.setdefault(i, oi)
    scratch = {j: np.empty(CHUNK, dtype=np.dtype(dt)) for j, (_, _, dt) in enumerate(prog.nodes) if j not in out_of}
    for start in range(0, size, CHUNK):
        stop = min(start + CHUNK, size)
        n = stop - start
        targets = {j: (out_flat[out_of[j]][start:stop] if j in out_of else scratch[j][:n])
                   for j in range(len(prog.nodes))}
        res = _program_eval(prog, [f[start:stop] for f in flats], targets)
        for oi, r in enumerate(res):
            if prog.outputs[oi][0] != "node" or out_of[prog.outputs[oi][1]] != oi:
                out_flat[oi][start:stop] = r
    return outs


def eval_composite(prog, inputs):
    """CompositeElemwise.perform dispatch (ops/elemwise.py:538-544)."""
    same = len({a.shape for a in inputs}) <= 1
    contig = all(a.flags["C_CONTIGUOUS"] for a in inputs)
    if inputs and same and contig and inputs[0].size >= CHUNK:
        return eval_composite_chunked(prog, inputs)
    return eval_composite_plain(prog, inputs)


# ---------------------------------------------------------------- interpreter

def _toposort(outputs):
    nodes, seen, stack = {}, set(), list(outputs)
    while stack:
        v = stack.pop()
        if v.id in seen:
            continue
        seen.add(v.id)
        if v.owner is not None and v.owner.id not in nodes:
            nodes[v.owner.id] = v.owner
            stack.extend(v.owner.inputs)
    indeg, succ = {}, {i: [] for i in nodes}
    for n in nodes.values():
        preds = {x.owner.id for x in n.inputs if x.owner is not None}
        indeg[n.id] = len(preds)
        for p in preds:
            succ[p].append(n.id)
    heap = [i for i, d in indeg.items() if d == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        i = heapq.heappop(heap)
        order.append(nodes[i])
        for s in succ[i]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(heap, s)
    return order


def run_node(node, args):
    op = node.op
    name = op.name
    if name == "elemwise":
        return [elemwise(op.kernel, args)]
    if name == "composite":
        return eval_composite(op.program, args)
    if name == "sum":
        return [reduce_sum(args[0], op.axes)]
    if name == "max":
        return [reduce_max(args[0], op.axes)]
    if name == "argmax_onehot":
        return [argmax_onehot(args[0], op.axes)]
    if name == "argmax":
        return [argmax_index(args[0], op.axes)]
    if name == "dot":
        return [dot(*args)]
    if name == "dot_epilogue":  # the device's fused form of dot + its consumer
        z = dot(args[0], args[1])
        if op.kind == 7:
            return [elemwise("add", [args[3], elemwise("add", [args[2], z])])]
        if op.kind == 1:
            return [elemwise("add", [args[2], z])]
        if op.kind == 4:
            h = elemwise("tanh", [elemwise("add", [args[2], z])])
            return [h, elemwise("sub", [np.asarray(1, dtype=h.dtype), elemwise("sqr", [h])])]
        return [elemwise("mul", [z, args[2]])]
    if name == "dimshuffle":
        return [dimshuffle(args[0], op.pattern)]
    if name == "subtensor":
        return [subtensor(args[0], op.items)]
    if name == "inc_subtensor":
        return [inc_subtensor(args[0], args[1], op.items)]
    if name == "join":
        return [join(op.axis, args)]
    if name == "shape_of":
        return [np.asarray(np.shape(args[0]), dtype=np.int64)]
    if name == "reshape":
        return [reshape(args[0], args[1])]
    if name == "scan":
        return scan_loop(op, args)
    if name == "zero_embed":  # device rewrite of the inc_subtensor chain over zeros_like it replaces
        out = np.zeros(np.shape(args[0]), dtype=np.asarray(args[0]).dtype)
        for items, v in zip(op.regions, args[1:]):
            out[_as_index(items)] += v
        return [out]
    raise NotImplementedError(f"oracle has no kernel for op {name!r}")


def reshape(x, shp):
    """Reshape.perform (ops/shaping.py:333-338): np.reshape, ShapeMismatch on failure."""
    try:
        return np.reshape(x, tuple(int(s) for s in shp))
    except ValueError as exc:
        from paper_1605_02688_b200.errors import ShapeMismatch
        raise ShapeMismatch(f"reshape: {exc}") from exc


def scan_loop(op, args):
    """ScanOp.perform (scan.py:248-300): outer inputs [n_steps?, sequences,
    initial states, invariants]; every step evaluates the inner graph on
    [sequence elements, states, invariants]; outputs are the histories of
    every inner output (the whole sequence, or only the last step for
    retention "last") followed by each state's final value.  A zero-length
    loop probes the inner graph once (on ones) for the history shapes."""
    from paper_1605_02688_b200.errors import LengthMismatch
    pos = 1 if op.has_nsteps else 0
    seqs = [np.asarray(a) for a in args[pos: pos + op.n_seqs]]
    states = [np.asarray(a) for a in args[pos + op.n_seqs: pos + op.n_seqs + op.n_states]]
    nonseqs = [np.asarray(a) for a in args[pos + op.n_seqs + op.n_states:]]
    lengths = {int(q.shape[0]) for q in seqs}
    if len(lengths) > 1:
        raise LengthMismatch(f"sequences disagree on length: {sorted(lengths)}")
    if op.has_nsteps:
        length = int(args[0])
        if length < 0:
            raise LengthMismatch(f"negative step count {length}")
        if lengths and length != next(iter(lengths)):
            raise LengthMismatch(f"step count {length} != shared sequence length {next(iter(lengths))}")
    elif lengths:
        length = next(iter(lengths))
    else:
        raise LengthMismatch("loop without sequences needs an explicit step count")
    inner = list(op.inner_inputs)

    def step(vals):
        return evaluate(list(op.inner_outputs), dict(zip(inner, vals)))
    full = [r == "full" for r in op.retention]
    if length == 0:
        probe = [np.ones(q.shape[1:], dtype=q.dtype) for q in seqs] + states + nonseqs
        hist = [np.zeros((0,) + np.shape(o), dtype=np.dtype(v.type.dtype))
                for o, v in zip(step(probe), op.inner_outputs)]
        return hist + [np.array(x, copy=True) for x in states]
    steps = []
    for t in range(length):
        outs = step([q[t] for q in seqs] + states + nonseqs)
        outs = [np.asarray(o, dtype=np.dtype(v.type.dtype)) for o, v in zip(outs, op.inner_outputs)]
        steps.append(outs)
        states = [np.array(outs[k], copy=True) for k in range(op.n_states)]
    hist = []
    for i in range(len(op.inner_outputs)):
        if full[i]:
            hist.append(np.stack([s[i] for s in steps]))
        else:
            hist.append(np.asarray(steps[-1][i])[None])
    return hist + [np.array(x, copy=True) for x in states]


def _as_index(items):
    """ops/shaping.py _as_index: ints stay, (start, stop, step) triples are slices."""
    return tuple(i if isinstance(i, int) else slice(*i) for i in items)


def subtensor(x, items):
    """Subtensor.perform (ops/shaping.py:157-162): basic slicing, a view."""
    return x[_as_index(items)]


def inc_subtensor(target, value, items):
    """IncSubtensor.perform (ops/shaping.py:238-242): a copy of target with
    value added into the region."""
    out = target.copy()
    out[_as_index(items)] += value
    return out


def join(axis, xs):
    """Join.perform (ops/shaping.py:416-420): np.concatenate along axis."""
    return np.concatenate(xs, axis=axis)


def evaluate(outputs, bindings):
    """interp.eval_graph (interp.py:20-51): topological walk, one host kernel
    per node, values cast to the declared dtype on binding."""
    env = {}
    for var, val in bindings.items():
        env[var.id] = np.asarray(val, dtype=np.dtype(var.type.dtype))
    for node in _toposort(outputs):
        args = []
        for x in node.inputs:
            if x.id in env:
                args.append(env[x.id])
            elif hasattr(x, "value"):
                args.append(x.value)
            elif hasattr(x, "get_value"):
                args.append(x.get_value())
            else:
                raise KeyError(f"oracle: no value bound for {x!r}")
        for o, r in zip(node.outputs, run_node(node, args)):
            env[o.id] = np.asarray(r)
    res = []
    for o in outputs:
        if o.id in env:
            res.append(env[o.id])
        elif hasattr(o, "value"):
            res.append(np.asarray(o.value))
        else:
            res.append(np.asarray(o.get_value()))
    return res


def evaluate_order(order, outputs, bindings, after_node=None):
    """Like ``evaluate`` but over a given node order, calling
    ``after_node(node, values)`` after each node (the data-parallel test uses
    it to allreduce partial sums exactly where the device step does)."""
    env = {var.id: np.asarray(val, dtype=np.dtype(var.type.dtype)) for var, val in bindings.items()}
    for node in order:
        args = [env[x.id] if x.id in env else np.asarray(x.value) for x in node.inputs]
        res = [np.asarray(r) for r in run_node(node, args)]
        if after_node is not None:
            res = after_node(node, res) or res
        for o, r in zip(node.outputs, res):
            env[o.id] = r
    return [env[o.id] if o.id in env else np.asarray(o.value) for o in outputs]
