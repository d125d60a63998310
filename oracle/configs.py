"""The five BASELINE configs as graphs (SURVEY Appendix A recipes), plus
their seeded synthetic inputs.  Test / bench infrastructure.

``build_*`` return graph pieces built with the product's symbolic front end
(the same spelling a reference user writes); ``inputs_*`` return the NumPy
inputs; ``cpu_*`` evaluate a config with the oracle kernels in
``texpr_numpy`` — the CPU reference path timed beside the GPU.
"""
from __future__ import annotations

import numpy as np

F32 = "float32"


def softmax_xent_cost(T, z, y, n_global):
    from paper_1605_02688_b200.ops import dimshuffle
    m = T.max(z, axis=1)
    e = T.exp(z - dimshuffle(m, (0, "x")))
    p = e / dimshuffle(T.sum(e, axis=1), (0, "x"))
    return -T.sum(y * T.log(p)) / float(n_global)


# ---------------------------------------------------------------- config 1
def inputs_logreg(N=600, D=784, K=10, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.random((N, D), dtype=np.float32)
    y = np.eye(K, dtype=np.float32)[rng.integers(0, K, N)]
    return x, y


def build_logreg(T, N=600, D=784, K=10, lr=0.13):
    x, y = T.matrix("x", dtype=F32), T.matrix("y", dtype=F32)
    W = T.shared(np.zeros((D, K), np.float32), name="W")
    b = T.shared(np.zeros(K, np.float32), name="b")
    cost = softmax_xent_cost(T, T.dot(x, W) + b, y, N)
    gW, gb = T.grad(cost, [W, b])
    return dict(inputs=[x, y], outputs=[cost], updates=[(W, W - lr * gW), (b, b - lr * gb)], params=[W, b])


# ---------------------------------------------------------------- config 2
def inputs_ew(n=1 << 28, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(n, dtype=np.float32) for _ in range(4)]


def build_ew(T):
    a, b, c, d = (T.vector(s, dtype=F32) for s in "abcd")
    return dict(inputs=[a, b, c, d], outputs=T.sigmoid(a * b + c) ** 2 - d)


# ---------------------------------------------------------------- config 3
def inputs_reduce(n=16384, seed=0):
    return np.random.default_rng(seed).standard_normal((n, n), dtype=np.float32)


# ---------------------------------------------------------------- configs 4/5
def init_mlp_params(D=784, H=4096, K=10, seed=0):
    rng = np.random.default_rng(seed)
    Ws = [(rng.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32) for i, o in ((D, H), (H, H), (H, K))]
    bs = [np.zeros(H, np.float32), np.zeros(H, np.float32), np.zeros(K, np.float32)]
    return Ws, bs


def build_mlp(T, B=8192, D=784, H=4096, K=10, lr=0.01, seed=0, n_global=None):
    Ws, bs = init_mlp_params(D, H, K, seed)
    x, y = T.matrix("x", dtype=F32), T.matrix("y", dtype=F32)
    W1, W2, W3 = (T.shared(w, name=f"W{i + 1}") for i, w in enumerate(Ws))
    b1, b2, b3 = (T.shared(b, name=f"b{i + 1}") for i, b in enumerate(bs))
    h1 = T.tanh(T.dot(x, W1) + b1)
    h2 = T.tanh(T.dot(h1, W2) + b2)
    cost = softmax_xent_cost(T, T.dot(h2, W3) + b3, y, n_global or B)
    params = [W1, b1, W2, b2, W3, b3]
    grads = T.grad(cost, params)
    return dict(inputs=[x, y], outputs=[cost], updates=[(p, p - lr * g) for p, g in zip(params, grads)],
                params=params)


def inputs_mlp(B=8192, D=784, K=10, seed=1):
    rng = np.random.default_rng(seed)
    x = rng.random((B, D), dtype=np.float32)
    y = np.eye(K, dtype=np.float32)[rng.integers(0, K, B)]
    return x, y


# ---------------------------------------------------------------- CPU path

class CpuFunction:
    """The reference's compiled function restated on the oracle kernels:
    same rewrite preset (so the same node list), NumPy per node, updates
    written back after the walk (runtime.py:375-426)."""

    def __init__(self, T, inputs, outputs, updates=(), preset="fast_run", exclude=()):
        from paper_1605_02688_b200.graph import FunctionGraph, Variable, clone_outputs
        from paper_1605_02688_b200.rewrite import run_preset
        from paper_1605_02688_b200.shared import SharedVariable
        single = not isinstance(outputs, (list, tuple))
        outs = [outputs] if single else list(outputs)
        self.single = single
        self.updates = list(updates)
        uvals = [u for _, u in self.updates]
        found, seen, stack = [], set(), outs + uvals
        stack = list(stack)
        while stack:
            v = stack.pop()
            if v.id in seen or any(v is i for i in inputs):
                continue
            seen.add(v.id)
            if v.owner is not None:
                stack.extend(v.owner.inputs)
            elif isinstance(v, SharedVariable):
                found.append(v)
        found.sort(key=lambda v: v.id)
        self.shared = found
        full = list(inputs) + found
        repl = {v: Variable(v.type, v.name) for v in full}
        cloned, _ = clone_outputs(outs + uvals, repl)
        self.fg = FunctionGraph([repl[v] for v in full], cloned)
        # the reference has no GEMM epilogues: keep its node list
        run_preset(self.fg, preset, exclude=tuple(exclude) + (
            "fuse_gemm_epilogue", "fuse_narrow_grad", "loop_pushout_sequences", "loop_pushout_accumulators",
            "loop_pushout_outputs", "loop_drop_unused_outputs", "add_into_zero_inc", "loop_body_zero_inc_chains"))
        self.in_vars = [repl[v] for v in inputs]
        self.sh_vars = [repl[v] for v in found]
        self.n_out = len(outs)
        self.values = {id(s): s.get_value() for s in found}
        self.node_time = 0.0

    def __call__(self, *vals):
        import time
        from oracle import texpr_numpy as O
        bind = {v: np.array(x, dtype=np.dtype(v.type.dtype), copy=True) for v, x in zip(self.in_vars, vals)}
        for s, v in zip(self.shared, self.sh_vars):
            bind[v] = self.values[id(s)]
        t0 = time.perf_counter()
        res = O.evaluate(self.fg.outputs, bind)
        self.node_time += time.perf_counter() - t0
        outs = [np.array(r, copy=True) for r in res[: self.n_out]]
        for (s, _), r in zip(self.updates, res[self.n_out:]):
            self.values[id(s)] = np.array(r, copy=True)
        return outs[0] if self.single else outs

    def value(self, s):
        return self.values[id(s)]
