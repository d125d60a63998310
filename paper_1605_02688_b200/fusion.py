"""Convex elementwise fusion (stage ``specialize``, name ``fuse_elemwise``).

Replaces reference ``rewrites/fusion.py:47-144``, whose union-find joins every
elementwise producer/consumer edge without a convexity check and therefore
raises ``CycleDetected`` on any graph where a reduction or dot sits between
two elementwise nodes of one group (SURVEY F2 — both training configs).

Here groups grow greedily in topological order and a node joins its
producer's group only if (a) its output has the group's iteration space
(same rank and broadcast pattern, so one generated kernel covers every member)
and (b) no path leaves the group and re-enters at the node (convexity),
checked against per-node ancestor sets.  Each group of >= 2 nodes becomes one
``Composite`` whose program is the NVRTC cache key; values consumed outside the
group become extra kernel outputs; 0-d and single-element constants are
inlined as literals.
"""
from __future__ import annotations

from .elemwise import Composite, Elemwise, EwProgram
from .errors import CycleDetected
from .graph import Constant, apply
from .rewrite import register_rewrite


def _fusable(node) -> bool:
    return isinstance(node.op, (Elemwise, Composite)) and len(node.outputs) >= 1


def _space(node):
    t = node.outputs[0].type
    if any(o.type.broadcastable != t.broadcastable for o in node.outputs):
        return None
    return t.broadcastable


def _inline(x) -> bool:
    return isinstance(x, Constant) and x.value.size == 1


@register_rewrite("fuse_elemwise", "specialize", "global")
def fuse_elemwise(fgraph, ctx, emit) -> int:
    order = fgraph.toposort()
    anc: dict[int, frozenset] = {}
    for n in order:
        s = set()
        for x in n.inputs:
            if x.owner is not None and x.owner.id in fgraph.nodes:
                s.add(x.owner.id)
                s |= anc[x.owner.id]
        anc[n.id] = frozenset(s)

    group_of: dict[int, int] = {}
    members: dict[int, list] = {}
    for n in order:
        if not _fusable(n) or _space(n) is None:
            continue
        joined = None
        for x in n.inputs:
            p = x.owner
            if p is None or p.id not in group_of:
                continue
            g = group_of[p.id]
            if _space(members[g][0]) != _space(n):
                continue
            gset = {m.id for m in members[g]}
            ok = True
            for y in n.inputs:
                q = y.owner
                if q is None or q.id in gset:
                    continue
                if anc[q.id] & gset:  # a path leaves the group and comes back
                    ok = False
                    break
            if ok:
                joined = g
                break
        if joined is None:
            group_of[n.id] = n.id
            members[n.id] = [n]
        else:
            group_of[n.id] = joined
            members[joined].append(n)

    applied = 0
    for root in sorted(members):
        grp = members[root]
        if len(grp) >= 2:
            applied += _fuse_capped(fgraph, grp, emit)
    return applied


MAX_OPERANDS = 24  # generated kernel signature limit (codegen.generate_source)


def _operands(fgraph, grp) -> int:
    ids = {n.id for n in grp}
    produced = {o.id for n in grp for o in n.outputs}
    leaves = {x.id for n in grp for x in n.inputs if x.id not in produced and not _inline(x)}
    boundary = sum(1 for n in grp for o in n.outputs
                   if fgraph.is_output(o) or any(c.id not in ids for c in fgraph.node_clients(o)))
    return len(leaves) + boundary


def _fuse_capped(fgraph, grp, emit) -> int:
    """Fuse a convex group; a group needing more kernel operands than the
    generator supports is split at its topological midpoint (a prefix and the
    matching suffix of a convex group are both convex and cannot form a
    cycle with each other).  Groups are convex individually, but two groups
    can still depend on each other through members of both (a1 -> b1 and
    b2 -> a2); fusing the second would then close a cycle, so that group stays
    unfused (``replace_all`` is transactional and reports it)."""
    from .errors import CycleDetected
    if len(grp) < 2:
        return 0
    if _operands(fgraph, grp) > MAX_OPERANDS:
        half = len(grp) // 2
        return _fuse_capped(fgraph, grp[:half], emit) + _fuse_capped(fgraph, grp[half:], emit)
    try:
        return 1 if _fuse(fgraph, grp, emit) else 0
    except CycleDetected:
        return 0


def _fuse(fgraph, grp, emit) -> bool:
    ids = {n.id for n in grp}
    produced = {o.id for n in grp for o in n.outputs}
    leaves, leaf_pos = [], {}
    consts, const_pos = [], {}
    for n in grp:
        for x in n.inputs:
            if x.id in produced:
                continue
            if _inline(x):
                key = (x.type.dtype, x.value.reshape(()).item())
                if key not in const_pos:
                    const_pos[key] = len(consts)
                    consts.append(key)
            elif x.id not in leaf_pos:
                leaf_pos[x.id] = len(leaves)
                leaves.append(x)
    boundary = []
    for n in grp:
        for o in n.outputs:
            if fgraph.is_output(o) or any(c.id not in ids for c in fgraph.node_clients(o)):
                boundary.append(o)
    if not boundary:
        return False

    refs: dict[int, tuple] = {}
    prog_nodes = []

    def ref_of(x):
        if x.id in refs:
            return refs[x.id]
        if x.id in leaf_pos:
            return ("in", leaf_pos[x.id])
        return ("const", const_pos[(x.type.dtype, x.value.reshape(()).item())])

    for n in grp:
        if isinstance(n.op, Elemwise):
            prog_nodes.append((n.op.kernel, [ref_of(x) for x in n.inputs], n.outputs[0].type.dtype))
            refs[n.outputs[0].id] = ("node", len(prog_nodes) - 1)
        else:  # splice an inner Composite's program
            p = n.op.program
            local = {}
            outer_in = [ref_of(x) for x in n.inputs]
            for j, (k, rr, dt) in enumerate(p.nodes):
                mapped = []
                for kind, i in rr:
                    if kind == "in":
                        mapped.append(outer_in[i])
                    elif kind == "node":
                        mapped.append(local[i])
                    else:
                        key = p.consts[i]
                        if key not in const_pos:
                            const_pos[key] = len(consts)
                            consts.append(key)
                        mapped.append(("const", const_pos[key]))
                prog_nodes.append((k, mapped, dt))
                local[j] = ("node", len(prog_nodes) - 1)
            for o, r in zip(n.outputs, p.outputs):
                refs[o.id] = local[r[1]] if r[0] == "node" else (
                    outer_in[r[1]] if r[0] == "in" else r)

    prog = EwProgram([x.type.dtype for x in leaves], consts, prog_nodes, [refs[b.id] for b in boundary])
    outs = apply(Composite(prog), leaves)
    if any(o.type != b.type for o, b in zip(outs, boundary)):
        return False
    fgraph.replace_all(list(zip(boundary, outs)), "fuse_elemwise")
    emit(node=grp[-1], replaced=f"group[{len(grp)}]", replacement=outs[0].owner.op.display_name)
    return True


# ---------------------------------------------------------------------------
# GEMM epilogue fusion (stage abstract_select, after elementwise fusion)

def _match_bias_tanh_dual(prog, z_idx):
    """{t0 = add(b, z); t1 = tanh(t0); t2 = sqr(t1); t3 = sub(1, t2)} with
    outputs (t1, t3) — the MLP layer's forward Composite (tanh and the
    1 - h^2 factor its gradient needs)."""
    nodes = prog.nodes
    if len(nodes) != 4 or len(prog.in_dtypes) != 2 or prog.outputs != (("node", 1), ("node", 3)):
        return False
    (k0, r0, _), (k1, r1, _), (k2, r2, _), (k3, r3, _) = nodes
    b_idx = 1 - z_idx
    if k0 != "add" or set(r0) != {("in", z_idx), ("in", b_idx)}:
        return False
    if k1 != "tanh" or r1 != (("node", 0),) or k2 != "sqr" or r2 != (("node", 1),):
        return False
    if k3 != "sub" or r3[1] != ("node", 2) or r3[0][0] != "const":
        return False
    return float(prog.consts[r3[0][1]][1]) == 1.0


_NO_AUX_BIAS = bool(__import__("os").environ.get("TX_FUSE_NO_AUX_BIAS"))  # A/B diagnostic


def _match_add_aux_bias(prog, z_idx):
    """{t0 = add(g, z); t1 = add(b, t0)} with output t1, g a second [M,N]
    operand and b a row: a recurrent layer's pre-activation
    (x-projection + h.W + bias).  Returns (g index, b index) or None."""
    nodes = prog.nodes
    if len(nodes) != 2 or len(prog.in_dtypes) != 3 or prog.outputs != (("node", 1),):
        return None
    (k0, r0, _), (k1, r1, _) = nodes
    if k0 != "add" or k1 != "add" or ("in", z_idx) not in r0 or ("node", 0) not in r1:
        return None
    g = [r for r in r0 if r != ("in", z_idx)]
    b = [r for r in r1 if r != ("node", 0)]
    if len(g) != 1 or len(b) != 1 or g[0][0] != "in" or b[0][0] != "in" or g[0][1] == b[0][1]:
        return None
    return g[0][1], b[0][1]


def _sole_dot_client(fgraph, z, Dot):
    """z = dot(a, b) feeding exactly one consumer (and not a graph output)."""
    if z.owner is None or not isinstance(z.owner.op, Dot) or fgraph.is_output(z):
        return False
    a, b = z.owner.inputs
    return a.type.ndim == 2 and b.type.ndim == 2 and len(fgraph.node_clients(z)) == 1 \
        and len(fgraph.clients[z]) == 1


def _fuse_tanh_layers(fgraph, emit) -> int:
    """Forward layer h = tanh(b + x.W) whose 1 - h^2 only feeds backward
    products mul(dz.W^T, 1 - h^2): emit dot+bias_tanh for h and
    dot+mul_1msqr(h) for each backward product, so 1 - h^2 is never
    materialised (one [B,H] store and one [B,H] load fewer per layer than the
    dual-output form).  Same scalar ops and rounding order as the unfused
    nodes (sqr, sub(1, .), mul)."""
    from .linalg import EPI_BIAS_TANH, EPI_MUL_1MSQR, Dot, DotEpilogue
    applied = 0
    for c in list(fgraph.toposort()):
        if c.id not in fgraph.nodes or not isinstance(c.op, Composite) or len(c.inputs) != 2:
            continue
        zi = next((i for i, x in enumerate(c.inputs) if _sole_dot_client(fgraph, x, Dot)), None)
        if zi is None:
            continue
        z, bias = c.inputs[zi], c.inputs[1 - zi]
        if bias is z or bias.type.ndim != 1 or bias.type.dtype != z.type.dtype \
                or not _match_bias_tanh_dual(c.op.program, zi):
            continue
        h, g = c.outputs
        users = fgraph.node_clients(g)
        if fgraph.is_output(g) or not users:
            continue
        back = []
        for m in users:
            if not (isinstance(m.op, Elemwise) and m.op.kernel == "mul" and len(m.inputs) == 2):
                break
            z2 = m.inputs[1] if m.inputs[0] is g else m.inputs[0]
            if z2 is g or z2.type != g.type or not _sole_dot_client(fgraph, z2, Dot) \
                    or m.outputs[0].type != z2.type:
                break
            back.append((m, z2))
        else:
            a, b = z.owner.inputs
            (hn,) = apply(DotEpilogue(EPI_BIAS_TANH), [a, b, bias])
            if hn.type != h.type:
                continue
            repl = [(h, hn)]
            for m, z2 in back:
                a2, b2 = z2.owner.inputs
                (o,) = apply(DotEpilogue(EPI_MUL_1MSQR), [a2, b2, hn])
                repl.append((m.outputs[0], o))
            fgraph.replace_all(repl, "fuse_gemm_epilogue")
            emit(node=c, replaced="dot+composite[tanh,1-h^2]", replacement=f"dot+bias_tanh + {len(back)} dot+mul_1msqr")
            applied += 1 + len(back)
    return applied


def _match_sgd(prog, z_idx):
    """{t0 = mul(lr, z); t1 = sub(w, t0)} with output t1 (either operand
    order of the mul): the SGD update w - lr * grad.  Returns lr or None."""
    if len(prog.nodes) != 2 or len(prog.in_dtypes) != 2 or prog.outputs != (("node", 1),):
        return None
    (k0, r0, _), (k1, r1, _) = prog.nodes
    if k0 != "mul" or k1 != "sub" or r1 != (("in", 1 - z_idx), ("node", 0)):
        return None
    others = [r for r in r0 if r != ("in", z_idx)]
    if len(r0) != 2 or len(others) != 1 or others[0][0] != "const":
        return None
    dt, val = prog.consts[others[0][1]]
    return float(val), dt


def _fuse_sgd_updates(fgraph, ctx, emit) -> int:
    """w - lr * dot(a, b) (a weight's SGD step from its gradient GEMM) becomes
    one GEMM whose epilogue reads w and writes the new w -- in place when the
    update can be written directly (the dW matrix is never stored).  Skipped
    for data-parallel steps, where the gradient is a partial sum that must be
    all-reduced before the update."""
    from .linalg import EPI_SGD, Dot, DotEpilogue
    if getattr(ctx, "data_parallel", False):
        return 0
    applied = 0
    for c in list(fgraph.toposort()):
        if c.id not in fgraph.nodes or not isinstance(c.op, Composite) or len(c.inputs) != 2:
            continue
        zi = next((i for i, x in enumerate(c.inputs) if _sole_dot_client(fgraph, x, Dot)), None)
        if zi is None:
            continue
        z, w = c.inputs[zi], c.inputs[1 - zi]
        if w is z or w.type != z.type or c.outputs[0].type != z.type:
            continue
        m = _match_sgd(c.op.program, zi)
        if m is None:
            continue
        a, b = z.owner.inputs
        (o,) = apply(DotEpilogue(EPI_SGD, m[0], m[1]), [a, b, w])
        fgraph.replace_all([(c.outputs[0], o)], "fuse_gemm_epilogue")
        emit(node=c, replaced="dot+composite[sgd]", replacement="dot+sgd")
        applied += 1
    return applied


def _fuse_narrow_grads(fgraph, emit) -> int:
    """Backward of a tanh layer h feeding a narrow layer: the three nodes
    that each stream a [B,H] tensor --
        dh = dot+mul_1msqr(dz, wt, h)          (dz [B,k], k small)
        gW = dot(h^T, dz)  or  dot+sgd(h^T, dz, w)
        db = sum[0](dh)                         (optional)
    -- become one narrow_grad node (one read of h, one write of dh)."""
    from .linalg import EPI_MUL_1MSQR, EPI_SGD, Dot, DotEpilogue, NarrowLayerGrad
    from .reduce import Sum
    from .shaping import DimShuffle
    applied = 0
    for o in list(fgraph.toposort()):
        if o.id not in fgraph.nodes or not (isinstance(o.op, DotEpilogue) and o.op.kind == EPI_MUL_1MSQR):
            continue
        dz, wt, h = o.inputs
        if dz.type.ndim != 2 or wt.type.ndim != 2 or dz.type.dtype != h.type.dtype:
            continue
        k = None
        for c in fgraph.node_clients(dz):
            if c is o or len(c.inputs) < 2 or c.inputs[1] is not dz or not c.inputs[0].owner:
                continue
            t = c.inputs[0].owner
            if not (isinstance(t.op, DimShuffle) and t.op.pattern == (1, 0) and t.inputs[0] is h):
                continue
            if type(c.op) is Dot or (isinstance(c.op, DotEpilogue) and c.op.kind == EPI_SGD):
                k = c
                break
        if k is None:
            continue
        dh = o.outputs[0]
        s = next((c for c in fgraph.node_clients(dh) if isinstance(c.op, Sum) and tuple(c.op.axes) == (0,)), None)
        sgd = isinstance(k.op, DotEpilogue)
        op = NarrowLayerGrad(sgd, k.op.alpha if sgd else 0.0, k.op.alpha_dtype if sgd else "float32", s is not None)
        outs = apply(op, [dz, wt, h] + ([k.inputs[2]] if sgd else []))
        old = [dh, k.outputs[0]] + ([s.outputs[0]] if s is not None else [])
        if [v.type for v in outs] != [v.type for v in old]:
            continue
        try:
            fgraph.replace_all(list(zip(old, outs)), "fuse_gemm_epilogue")
        except CycleDetected:
            continue
        emit(node=o, replaced="dot+mul_1msqr, " + getattr(k.op, "display_name", k.op.name)
             + (", sum[0]" if s is not None else ""), replacement=op.display_name)
        applied += 1
    return applied


@register_rewrite("fuse_gemm_epilogue", "abstract_select", "global")
def fuse_gemm_epilogue(fgraph, ctx, emit) -> int:
    from .linalg import EPI_ADD_AUX_BIAS, EPI_BIAS, EPI_BIAS_TANH_DUAL, EPI_MUL_AUX, Dot, DotEpilogue
    applied = _fuse_tanh_layers(fgraph, emit) + _fuse_sgd_updates(fgraph, ctx, emit)
    for d in list(fgraph.toposort()):
        if d.id not in fgraph.nodes or not isinstance(d.op, Dot):
            continue
        z = d.outputs[0]
        a, b = d.inputs
        if a.type.ndim != 2 or b.type.ndim != 2 or z.type.dtype not in ("float32", "float64"):
            continue
        if fgraph.is_output(z):
            continue
        clients = fgraph.node_clients(z)
        if len(clients) != 1 or len(fgraph.clients[z]) != 1:
            continue
        c = clients[0]
        kind, aux, extra = None, None, []
        if isinstance(c.op, Composite) and len(c.inputs) == 3 and z in c.inputs and c.inputs.count(z) == 1 \
                and not _NO_AUX_BIAS:
            m = _match_add_aux_bias(c.op.program, c.inputs.index(z))
            if m is not None:
                g, bias = c.inputs[m[0]], c.inputs[m[1]]
                if (g.type.dtype == bias.type.dtype == z.type.dtype and g.type.broadcastable == (False, False)
                        and bias.type.ndim == 1 and not bias.type.broadcastable[0]):
                    kind, aux, extra = EPI_ADD_AUX_BIAS, g, [bias]
        if isinstance(c.op, Composite) and len(c.inputs) == 2 and z in c.inputs:
            zi = c.inputs.index(z)
            other = c.inputs[1 - zi]
            if other is not z and other.type.ndim == 1 and other.type.dtype == z.type.dtype \
                    and _match_bias_tanh_dual(c.op.program, zi):
                kind, aux = EPI_BIAS_TANH_DUAL, other
        elif isinstance(c.op, Elemwise) and c.op.kernel in ("mul", "add") and len(c.inputs) == 2:
            other = c.inputs[1] if c.inputs[0] is z else c.inputs[0]
            if other is z or other.type.dtype != z.type.dtype:
                pass
            elif c.op.kernel == "mul" and other.type.broadcastable == z.type.broadcastable == (False, False):
                kind, aux = EPI_MUL_AUX, other
            elif c.op.kernel == "add" and other.type.ndim == 1 and not other.type.broadcastable[0]:
                kind, aux = EPI_BIAS, other
        if kind is None:
            continue
        outs = apply(DotEpilogue(kind), [a, b, aux] + extra)
        if [o.type for o in outs] != [o.type for o in c.outputs]:
            continue
        fgraph.replace_all(list(zip(c.outputs, outs)), "fuse_gemm_epilogue")
        emit(node=c, replaced=f"dot+{getattr(c.op, 'display_name', c.op.name)}", replacement=outs[0].owner.op.display_name)
        applied += 1
    return applied


@register_rewrite("fuse_narrow_grad", "abstract_select", "global")
def fuse_narrow_grad(fgraph, ctx, emit) -> int:
    """Runs after fuse_gemm_epilogue (registration order); separate so it can
    be excluded on its own (its gW / db sums run in a different order than
    the unfused kernels: equal within fp32 tolerance, not bitwise)."""
    return _fuse_narrow_grads(fgraph, emit)
