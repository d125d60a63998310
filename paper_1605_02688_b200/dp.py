"""Synchronous data parallelism for compiled training steps (config 5).

New subsystem; the paper's Platoon (``PAPER.md:530-546``) ran asynchronous
workers with host-memory parameters.  Here every GPU runs one process with the
same compiled step over its slice of the minibatch, parameters stay
replicated and device-resident, and the only exchange is an NCCL SUM
allreduce of the values the step computes as *partial sums* of the batch.

Which values are partial is derived, not declared: inputs marked sharded on
axis 0 are propagated through the optimized graph:

  * elementwise ops keep the shard axis (broadcast operands are replicated),
  * DimShuffle moves it, reductions/Dot that do not contract it keep it,
  * ``sum`` over the shard axis and ``dot`` contracting it produce PARTIAL
    values (the weight and bias gradients, and the cost's batch sum),
  * anything else touching the shard axis (max over the batch, ...) is
    rejected with NotSupported rather than silently computed per shard.

Each partial value is summed across ranks right after it is produced — so
every downstream node (the SGD updates) computes exactly what one GPU would
on the full batch, and replicas stay bit-identical.  Partial outputs are
packed into contiguous per-dtype buckets issued in production order on a
communication stream, overlapping the rest of the backward pass inside the
same captured CUDA graph.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .elemwise import Composite, Elemwise
from .errors import NotSupported
from .linalg import Dot
from .reduce import Sum, _Reduce
from .shaping import DimShuffle

REPLICATED = "R"
PARTIAL = "P"


def sharded(axis: int) -> str:
    return f"S{axis}"


def shard_axis(state):
    return int(state[1:]) if state and state[0] == "S" else None


@dataclass
class ShardPlan:
    state: dict = field(default_factory=dict)      # var id -> "R" | "P" | "S<k>"
    partial_nodes: list = field(default_factory=list)  # nodes whose outputs are allreduced, in order
    partial_vars: set = field(default_factory=set)     # ids of those outputs


def propagate(order, inputs_state: dict) -> ShardPlan:
    """Shard states for every variable of a scheduled graph."""
    st = dict(inputs_state)
    plan = ShardPlan(st)

    def get(v):
        return st.get(v.id, REPLICATED)

    for n in order:
        ins = [get(x) for x in n.inputs]
        op = n.op
        if all(s == REPLICATED for s in ins):
            for o in n.outputs:
                st[o.id] = REPLICATED
            continue
        rule = getattr(op, "shard_rule", None)
        if rule is not None:
            outs = rule(ins, sharded, PARTIAL, REPLICATED)
            if outs is None:
                raise NotSupported(f"{op.name}: no data-parallel rule for operand states {ins}")
            for o, s in zip(n.outputs, outs):
                if s == PARTIAL:
                    st[o.id] = REPLICATED  # reduced across ranks as soon as it is produced
                    plan.partial_vars.add(o.id)
                else:
                    st[o.id] = s
            if any(s == PARTIAL for s in outs):
                plan.partial_nodes.append(n)
            continue
        if isinstance(op, (Elemwise, Composite)):
            out_nd = n.outputs[0].type.ndim
            axes = set()
            for x, s in zip(n.inputs, ins):
                k = shard_axis(s)
                if k is not None:
                    axes.add(k + out_nd - x.type.ndim)
            if len(axes) != 1:
                raise NotSupported(f"{op.name}: operands sharded on different axes {sorted(axes)}")
            (ax,) = axes
            for o in n.outputs:
                st[o.id] = sharded(ax)
        elif isinstance(op, DimShuffle):
            k = shard_axis(ins[0])
            st[n.outputs[0].id] = sharded(op.pattern.index(k))
        elif isinstance(op, _Reduce):
            k = shard_axis(ins[0])
            if k in op.axes:
                if not isinstance(op, Sum):
                    raise NotSupported(f"{op.name} over the data-parallel axis needs a non-sum collective")
                st[n.outputs[0].id] = PARTIAL
                plan.partial_nodes.append(n)
            elif getattr(op, "name", "") == "argmax_onehot":
                st[n.outputs[0].id] = sharded(k)
            else:
                st[n.outputs[0].id] = sharded(k - sum(1 for a in op.axes if a < k))
        elif isinstance(op, Dot) or getattr(op, "gemm_operands", False):
            a, b = n.inputs[:2]
            ka, kb = shard_axis(ins[0]), shard_axis(ins[1])
            an = a.type.ndim
            if ka is not None and kb is not None:
                if not (ka == an - 1 and kb == 0):
                    raise NotSupported("dot: both operands sharded on non-contracted axes")
                out_state = PARTIAL
            elif ka is not None:
                if ka == an - 1:
                    raise NotSupported("dot: contraction over a sharded axis of one operand only")
                out_state = sharded(0)
            else:
                if kb == 0:
                    raise NotSupported("dot: contraction over a sharded axis of one operand only")
                out_state = sharded(n.outputs[0].type.ndim - 1)
            if len(n.inputs) > 2:  # fused GEMM epilogue operand (bias row or [M,N] factor)
                if out_state == PARTIAL:
                    raise NotSupported("a fused epilogue cannot act on a partial sum")
                se = ins[2]
                if se != REPLICATED and se != out_state:
                    raise NotSupported("dot epilogue operand sharded differently from the product")
            for o in n.outputs:
                st[o.id] = out_state
            if out_state == PARTIAL:
                plan.partial_nodes.append(n)
        else:
            raise NotSupported(f"op {op.name} has no data-parallel sharding rule")
        if n in plan.partial_nodes:
            # reduced across ranks as soon as it is produced: replicated downstream
            for o in n.outputs:
                st[o.id] = REPLICATED
                plan.partial_vars.add(o.id)
    return plan


class DataParallel:
    """One NCCL communicator over the processes of a torch.distributed group.

    ``shard_axis0``: which explicit inputs are split along axis 0 (default:
    all of them).  Create after ``torch.distributed.init_process_group``;
    with ``world_size=1`` it runs the same code path (allreduce on one rank).
    """

    def __init__(self, world_size: int | None = None, rank: int | None = None, shard_inputs=None,
                 bucket_bytes: int = 32 << 20, lib=None):
        import torch.distributed as dist
        if world_size is None:
            world_size = dist.get_world_size() if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank() if dist.is_initialized() else 0
        self.world_size, self.rank = world_size, rank
        self.shard_inputs = shard_inputs
        self.bucket_bytes = bucket_bytes
        self._lib = lib
        self._comm = None

    def comm(self, lib):
        if self._comm is None:
            uid = lib.nccl_unique_id() if self.rank == 0 else None
            if self.world_size > 1:
                import torch.distributed as dist
                box = [uid]
                dist.broadcast_object_list(box, src=0)
                uid = box[0]
            self._comm = lib.nccl_init(self.world_size, self.rank, uid)
        return self._comm

    def input_states(self, input_vars):
        out = {}
        for i, v in enumerate(input_vars):
            shard = self.shard_inputs is None or i in self.shard_inputs or v in (self.shard_inputs or ())
            if shard and v.type.ndim >= 1:
                out[v.id] = sharded(0)
        return out


def make_buckets(partials, bucket_bytes):
    """Group partial outputs into allreduce buckets.

    ``partials``: (var, nbytes, producer_pos, first_consumer_pos) in
    production order.  A bucket is one dtype, at most ``bucket_bytes`` (unless
    one tensor is larger), and never contains a value whose producer runs after
    another member's first consumer — so each bucket's allreduce can be issued
    before anything needs its result.
    """
    buckets, cur, cur_bytes, cur_dt, cur_need = [], [], 0, None, None
    for v, nbytes, prod, first_use in partials:
        dt = v.type.dtype
        if cur and (dt != cur_dt or cur_bytes + nbytes > bucket_bytes or (cur_need is not None and cur_need <= prod)):
            buckets.append(cur)
            cur, cur_bytes, cur_need = [], 0, None
        cur.append(v)
        cur_bytes += nbytes
        cur_dt = dt
        if first_use is not None:
            cur_need = first_use if cur_need is None else min(cur_need, first_use)
    if cur:
        buckets.append(cur)
    return buckets
