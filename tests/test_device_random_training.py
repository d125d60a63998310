"""Random training steps (grad + SGD updates) vs the reference algorithm.

Seeded random dense networks — 1 to 3 layers, tanh / sigmoid / rectifier
activations, widths and batch sizes that hit every GEMM path (skinny,
tcgen05, thin), softmax cross-entropy or squared-error loss, optional bias —
are compiled for the device with all device rewrites (GEMM epilogues, SGD
fusion, narrow-layer backward, row fusion) and stepped twice next to
``oracle.configs.CpuFunction`` (the reference's node list on NumPy kernels).

Tolerances: with ``gemm_mode="simt"`` (exact fp32 products) cost rtol 1e-5
and parameter relative L2 error 1e-5; with TF32 tensor-core GEMMs cost rtol
1e-3 and parameters 5e-3.
"""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C
from paper_1605_02688_b200.elemwise import make

pytestmark = pytest.mark.gpu


def _net(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.choice([33, 128, 300]))
    widths = [int(rng.choice([17, 64, 130]))]
    for _ in range(int(rng.integers(1, 4))):
        widths.append(int(rng.choice([10, 37, 64, 160])))
    acts = [str(rng.choice(["tanh", "sigmoid", "relu"])) for _ in widths[1:-1]]
    xent = bool(rng.random() < 0.6)
    bias = bool(rng.random() < 0.8)
    lr = float(rng.choice([0.01, 0.1]))
    x = T.matrix("x", dtype="float32")
    y = T.matrix("y", dtype="float32")
    params = []
    h = x
    for i, (a, b) in enumerate(zip(widths[:-1], widths[1:])):
        W = T.shared((rng.standard_normal((a, b)) / np.sqrt(a)).astype(np.float32), name=f"W{i}")
        params.append(W)
        z = T.dot(h, W)
        if bias:
            bv = T.shared((0.1 * rng.standard_normal(b)).astype(np.float32), name=f"b{i}")
            params.append(bv)
            z = z + bv
        if i < len(widths) - 2:
            act = acts[i]
            h = T.tanh(z) if act == "tanh" else T.sigmoid(z) if act == "sigmoid" else make("maximum", [z, 0.0])
        else:
            h = z
    if xent:
        m = T.max(h, axis=1)
        e = T.exp(h - T.dimshuffle(m, (0, "x")))
        p = e / T.dimshuffle(T.sum(e, axis=1), (0, "x"))
        cost = -T.sum(y * T.log(p)) / float(B)
        yv = np.eye(widths[-1], dtype=np.float32)[rng.integers(0, widths[-1], B)]
    else:
        d = h - y
        cost = T.sum(d * d) / float(B)
        yv = rng.standard_normal((B, widths[-1])).astype(np.float32)
    grads = T.grad(cost, params)
    updates = [(p_, p_ - lr * g) for p_, g in zip(params, grads)]
    xv = rng.standard_normal((B, widths[0])).astype(np.float32)
    return [x, y], [cost], updates, params, (xv, yv)


@pytest.mark.parametrize("mode,ctol,ptol", [("simt", 1e-5, 1e-5), ("auto", 1e-3, 5e-3)])
def test_random_training_steps_match_reference_algorithm(mode, ctol, ptol):
    for seed in range(24):
        ins, outs, ups, params, vals = _net(500 + seed)
        init = [p.get_value() for p in params]
        ref = C.CpuFunction(T, ins, outs, ups)
        want = [float(ref(*vals)[0]) for _ in range(2)]
        for p, v in zip(params, init):
            p.set_value(v)
        dev = T.compile(ins, outs, updates=ups, gemm_mode=mode)
        got = [float(dev(*vals)[0]) for _ in range(2)]
        for g, w in zip(got, want):
            assert abs(g - w) <= ctol * abs(w) + 1e-7, (seed, got, want)
        for (s, _), p in zip(ups, params):
            a, b = p.get_value(), ref.value(s)
            assert np.linalg.norm(a - b) <= ptol * max(np.linalg.norm(b), 1e-30), (seed, p.name)


def test_random_training_steps_data_parallel_single_rank():
    """The data-parallel path (sharding propagation, gradient buckets, NCCL
    allreduce inside the captured step) on one rank gives the plain step's
    results on random networks (row fusion off: then bit for bit)."""
    import os

    import torch.distributed as dist

    from paper_1605_02688_b200.dp import DataParallel
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    owns = not dist.is_initialized()
    if owns:
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for seed in range(12):
            ins, outs, ups, params, vals = _net(500 + seed)
            init = [p.get_value() for p in params]
            f = T.compile(ins, outs, updates=ups, row_fusion=False)
            ca = [float(f(*vals)[0]) for _ in range(2)]
            pa = [p.get_value() for p in params]
            for p, v in zip(params, init):
                p.set_value(v)
            g = T.compile(ins, outs, updates=ups, row_fusion=False, data_parallel=DataParallel(world_size=1, rank=0))
            cb = [float(g(*vals)[0]) for _ in range(2)]
            assert ca == cb, (seed, ca, cb)
            for p, a in zip(params, pa):
                assert np.array_equal(p.get_value(), a), (seed, p.name)
    finally:
        if owns:
            dist.destroy_process_group()
