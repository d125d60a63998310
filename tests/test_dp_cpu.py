"""Data-parallel step logic on CPU: sharding propagation finds exactly the
partial sums of the SURVEY §8(e) analysis, and a 2-rank gloo run that
allreduces them where the device step does reproduces the single-process
full-batch step (up to fp32 reassociation)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1605_02688_b200 as T
from oracle import configs as C
from oracle import texpr_numpy as O
from paper_1605_02688_b200 import dp
from paper_1605_02688_b200.errors import NotSupported

B, H = 64, 48


def _fn(B_local, n_global):
    g = C.build_mlp(T, B=B_local, H=H, n_global=n_global)
    f = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"], exclude=("fuse_elemwise",))
    return g, f


def test_propagation_finds_gradient_partials():
    g, f = _fn(B, B)
    order = f.fg.toposort()
    states = {v.id: dp.sharded(0) for v in f.in_vars}
    plan = dp.propagate(order, states)
    kinds = sorted(getattr(n.op, "display_name", n.op.name) for n in plan.partial_nodes)
    # dW1, dW2, dW3 (dot over the batch), db1, db2, db3 (sum[0]) and the cost's batch sum
    assert kinds == ["dot", "dot", "dot", "sum[0, 1]", "sum[0]", "sum[0]", "sum[0]"]
    for s, u in zip(g["params"], f.fg.outputs[1:]):
        assert plan.state[u.id] == dp.REPLICATED


def test_propagation_rejects_max_over_batch():
    x = T.matrix("x", dtype="float32")
    from paper_1605_02688_b200.graph import FunctionGraph
    fg = FunctionGraph([x], [T.max(x, axis=0)])
    with pytest.raises(NotSupported):
        dp.propagate(fg.toposort(), {x.id: dp.sharded(0)})


def test_buckets_respect_first_use():
    class V:
        def __init__(self, dt):
            self.type = type("t", (), {"dtype": dt})
    a, b, c = V("float32"), V("float32"), V("float32")
    # b is consumed (pos 5) before c is produced (pos 6): c starts a new bucket
    out = dp.make_buckets([(a, 10, 1, 9), (b, 10, 2, 5), (c, 10, 6, 9)], 1 << 20)
    assert [len(x) for x in out] == [2, 1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y = C.inputs_mlp(B=B)
        lo, hi = rank * B // world, (rank + 1) * B // world
        g, f = _fn(B // world, B)
        order = f.fg.toposort()
        plan = dp.propagate(order, {v.id: dp.sharded(0) for v in f.in_vars})
        partial = {n.id for n in plan.partial_nodes}

        def after(node, res):
            if node.id in partial:
                out = []
                for r in res:
                    t = torch.from_numpy(np.ascontiguousarray(r)).clone()
                    dist.all_reduce(t)
                    out.append(t.numpy())
                return out
        bind = {v: a for v, a in zip(f.in_vars, (x[lo:hi], y[lo:hi]))}
        for s, v in zip(f.shared, f.sh_vars):
            bind[v] = f.values[id(s)]
        res = O.evaluate_order(order, f.fg.outputs, bind, after)
        q.put((rank, float(res[0]), [np.asarray(r) for r in res[1:]]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_ranks_match_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda t: t[0])
    # replicas are bit-identical
    assert got[0][1] == got[1][1]
    for a, b in zip(got[0][2], got[1][2]):
        assert np.array_equal(a, b)
    # and equal the single-process full-batch step
    x, y = C.inputs_mlp(B=B)
    g, f = _fn(B, B)
    cost = f(x, y)[0]
    assert abs(got[0][1] - cost) <= 1e-6 * abs(cost)
    for (s, _), new in zip(g["updates"], got[0][2]):
        ref = f.value(s)
        assert np.linalg.norm(new - ref) <= 1e-6 * max(np.linalg.norm(ref), 1e-30)


def test_propagation_through_fused_gemm_epilogues():
    """With the device rewrites (GEMM epilogues), the same 7 partials."""
    from paper_1605_02688_b200.graph import FunctionGraph, Variable, clone_outputs
    from paper_1605_02688_b200.rewrite import RewriteContext, run_preset
    g = C.build_mlp(T, B=B, H=H)
    ins = g["inputs"] + g["params"]
    repl = {v: Variable(v.type, v.name) for v in ins}
    outs, _ = clone_outputs(g["outputs"] + [u for _, u in g["updates"]], repl)
    fg = FunctionGraph([repl[v] for v in ins], outs)
    # as compile(data_parallel=...) runs it: no SGD update fused into a partial-sum GEMM
    run_preset(fg, "fast_run", ctx=RewriteContext(execution_bound=True, data_parallel=True))
    names = [getattr(n.op, "display_name", n.op.name) for n in fg.toposort()]
    assert "dot+sgd" not in names
    assert names.count("dot+bias_tanh") == 2 and names.count("dot+mul_1msqr") == 0
    # each tanh layer's backward (dh, dW of the next layer, db) is one fused
    # node with two partial outputs
    assert names.count("narrow_grad+db") == 2
    plan = dp.propagate(fg.toposort(), {repl[v].id: dp.sharded(0) for v in g["inputs"]})
    assert len(plan.partial_nodes) == 5 and len(plan.partial_vars) == 7
    ng = next(n for n in fg.toposort() if n.op.name == "narrow_grad")
    assert plan.state[ng.outputs[0].id] == dp.sharded(0)
    assert {o.id for o in ng.outputs[1:]} <= plan.partial_vars
