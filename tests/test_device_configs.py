"""The BASELINE configs end to end on the device versus the reference's
goldens and the CPU oracle.

Tolerances: cost rtol 1e-3; parameters after SGD steps
||d-o||_2 / ||o||_2 <= 5e-3 (TF32 GEMMs); the logistic-
regression step runs only CUDA-core kernels (N = 10) and is held to 1e-5.
Full-size checks use size-independent properties (sampled indices for the
2^28 expression, exact max/argmax over the whole 16384^2 matrix).
"""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C
from oracle import texpr_numpy as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def test_logreg_three_steps_vs_reference(golden):
    x, y = C.inputs_logreg()
    g = C.build_logreg(T)
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    costs = np.array([step(x, y)[0] for _ in range(3)])
    np.testing.assert_allclose(costs, golden["cfg1_costs"], rtol=1e-5)
    assert abs(costs[0] - np.log(10)) < 1e-6
    W, b = g["params"]
    assert rel(W.get_value(), golden["cfg1_W"]) < 1e-5
    assert rel(b.get_value(), golden["cfg1_b"]) < 1e-5


def test_logreg_unfused_preset_matches():
    x, y = C.inputs_logreg()
    g = C.build_logreg(T)
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"], preset="fast_run", exclude=("fuse_elemwise",))
    assert len(step.order) == 44  # 45 reference nodes, the logits bias add folded into the GEMM
    g2 = C.build_logreg(T)
    fused = T.compile(g2["inputs"], g2["outputs"], updates=g2["updates"])
    for _ in range(3):
        a, b = step(x, y)[0], fused(x, y)[0]
        assert abs(a - b) <= 1e-6 * abs(b)


def test_mlp_small_vs_reference(golden):
    B, H = 64, 96
    g = C.build_mlp(T, B=B, H=H)
    x, y = C.inputs_mlp(B=B)
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    costs = np.array([step(x, y)[0] for _ in range(2)])
    np.testing.assert_allclose(costs, golden["cfg4_costs"], rtol=1e-3)
    for i, p in enumerate(g["params"]):
        assert rel(p.get_value(), golden[f"cfg4_p{i}"]) < 5e-3, i


def test_mlp_small_simt_mode_is_tight(golden):
    B, H = 64, 96
    g = C.build_mlp(T, B=B, H=H)
    x, y = C.inputs_mlp(B=B)
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"], gemm_mode="simt")
    costs = np.array([step(x, y)[0] for _ in range(2)])
    np.testing.assert_allclose(costs, golden["cfg4_costs"], rtol=1e-5)
    for i, p in enumerate(g["params"]):
        assert rel(p.get_value(), golden[f"cfg4_p{i}"]) < 1e-5, i


@pytest.mark.slow
def test_mlp_full_size_one_step_vs_oracle():
    B = 8192
    g = C.build_mlp(T, B=B)
    x, y = C.inputs_mlp(B=B)
    cpu = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"], exclude=("fuse_elemwise",))
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    c_dev = step(x, y)[0]
    c_ref = cpu(x, y)[0]
    assert abs(c_dev - c_ref) <= 1e-3 * abs(c_ref)
    for p in g["params"]:
        assert rel(p.get_value(), cpu.value(p)) < 5e-3, p.name


@pytest.mark.slow
def test_ew_full_size_sampled():
    n = 1 << 28
    g = C.build_ew(T)
    f = T.compile(g["inputs"], g["outputs"])
    ins = C.inputs_ew(n)
    out = f(*ins)
    idx = np.random.default_rng(1).integers(0, n, 1 << 16)
    want = O.eval_composite_plain(f.order[0].op.program, [a[idx] for a in ins])[0]
    np.testing.assert_allclose(out[idx], want, rtol=1e-5, atol=1e-6)
    assert np.isfinite(out).all()


@pytest.mark.slow
def test_reductions_full_size():
    X = C.inputs_reduce()
    v = T.matrix("X", dtype="float32")
    for ax in ((0,), (1,), (0, 1)):
        f = T.compile([v], [T.sum(v, axis=ax), T.max(v, axis=ax), T.argmax(v, axis=ax)])
        s, m, am = f(X)
        assert np.array_equal(m, O.reduce_max(X, ax))
        assert np.array_equal(am, O.argmax_index(X, ax))
        ref = O.reduce_sum(X, ax)
        bound = 2e-6 * (np.abs(X).sum(axis=ax) if len(ax) == 1 else np.abs(X).sum())
        assert np.all(np.abs(s - ref) <= bound)


def test_data_parallel_single_rank_matches_plain_step():
    """The DP path (sharding propagation, gradient buckets, NCCL allreduce
    captured in the step graph) on one rank equals the plain step bit-for-bit."""
    from paper_1605_02688_b200.dp import DataParallel
    B, H = 256, 512
    x, y = C.inputs_mlp(B=B)
    ga = C.build_mlp(T, B=B, H=H)
    fa = T.compile(ga["inputs"], ga["outputs"], updates=ga["updates"], row_fusion=False)
    gb = C.build_mlp(T, B=B, H=H)
    dp = DataParallel(world_size=1, rank=0, bucket_bytes=1 << 20)
    fb = T.compile(gb["inputs"], gb["outputs"], updates=gb["updates"], data_parallel=dp, row_fusion=False)
    # dW1..3, db1..3 and the cost's batch sum (the tanh layers' backward nodes carry two each)
    assert len(fb.shard.partial_vars) == 7
    for _ in range(3):
        ca, cb = fa(x, y)[0], fb(x, y)[0]
        assert ca == cb
    for pa, pb in zip(ga["params"], gb["params"]):
        assert np.array_equal(pa.get_value(), pb.get_value())
    # with row fusion the DP step keeps its partial sums outside the fused
    # blocks (their allreduce is scheduled); results agree to rounding
    gc = C.build_mlp(T, B=B, H=H)
    fc = T.compile(gc["inputs"], gc["outputs"], updates=gc["updates"],
                   data_parallel=DataParallel(world_size=1, rank=0))
    gd = C.build_mlp(T, B=B, H=H)
    fd = T.compile(gd["inputs"], gd["outputs"], updates=gd["updates"])
    for _ in range(3):
        cc, cd = fc(x, y)[0], fd(x, y)[0]
        assert abs(cc - cd) <= 1e-5 * abs(cd)


def test_row_fusion_matches_unfused_and_cuts_launches():
    x, y = C.inputs_logreg()
    ga = C.build_logreg(T)
    fa = T.compile(ga["inputs"], ga["outputs"], updates=ga["updates"], row_fusion=False)
    gb = C.build_logreg(T)
    fb = T.compile(gb["inputs"], gb["outputs"], updates=gb["updates"])
    for _ in range(4):
        ca, cb = fa(x, y)[0], fb(x, y)[0]
        assert abs(ca - cb) <= 1e-6 * abs(ca)
    for pa, pb in zip(ga["params"], gb["params"]):
        assert rel(pb.get_value(), pa.get_value()) < 1e-5
    plan = next(iter(fb._plans.values()))
    assert len(plan.row_groups) == 1
    assert len(plan.launches) <= 8 < len(next(iter(fa._plans.values())).launches)


def test_row_fusion_nan_and_ties_in_softmax_block():
    """max/argmax inside the fused block keep NumPy's NaN / first-index rules."""
    v = T.matrix("z", dtype="float32")
    m = T.max(v, axis=1)
    oh = T.argmax_onehot(v, axis=1)
    s = T.sum(T.exp(v - T.dimshuffle(m, (0, "x"))), axis=1)
    f = T.compile([v], [m, oh, s, T.argmax(v, axis=1)])
    z = np.random.default_rng(3).standard_normal((300, 37)).astype(np.float32)
    z[4, :] = 1.0
    z[7, 5] = np.nan
    z[9, 36] = np.nan
    z[9, 2] = np.nan
    got = f(z)
    assert len(next(iter(f._plans.values())).row_groups) == 1
    np.testing.assert_array_equal(got[0], O.reduce_max(z, (1,)))
    np.testing.assert_array_equal(got[1], O.argmax_onehot(z, (1,)))
    np.testing.assert_array_equal(got[3], O.argmax_index(z, (1,)))
    ref = O.reduce_sum(np.exp(z - O.reduce_max(z, (1,))[:, None]), (1,))
    np.testing.assert_allclose(got[2], ref, rtol=1e-5, equal_nan=True)


def test_gemm_epilogue_fusion_is_bit_exact():
    """dot+bias+tanh and dot*(1-h^2) (from the forward h) fused into the GEMM epilogues
    round exactly like the separate elementwise kernels."""
    B, H = 256, 512
    x, y = C.inputs_mlp(B=B)
    ga = C.build_mlp(T, B=B, H=H)
    fa = T.compile(ga["inputs"], ga["outputs"], updates=ga["updates"], exclude=("fuse_gemm_epilogue",))
    gb = C.build_mlp(T, B=B, H=H)
    fb = T.compile(gb["inputs"], gb["outputs"], updates=gb["updates"], exclude=("fuse_narrow_grad",))
    kinds = [getattr(n.op, "display_name", n.op.name) for n in fb.order]
    assert kinds.count("dot+bias_tanh") == 2 and kinds.count("dot+mul_1msqr") == 2
    for _ in range(2):
        assert fa(x, y)[0] == fb(x, y)[0]
    for pa, pb in zip(ga["params"], gb["params"]):
        assert np.array_equal(pa.get_value(), pb.get_value())


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,K", [(256, 512, 10), (1000, 1028, 7), (8192, 4096, 10), (96, 64, 16), (40, 36, 1)])
def test_narrow_grad_fusion_matches_unfused(B, H, K):
    """The fused narrow-layer backward (dh, dW of the narrow layer, db in one
    pass over h) equals the unfused dot+mul_1msqr / dot+sgd / sum[0] nodes
    within fp32 reassociation, and the hidden layer's wide case (fallback
    inside tx_narrow_grad) runs the same kernels as before."""
    x, y = C.inputs_mlp(B=B, D=64, K=K)
    ga = C.build_mlp(T, B=B, D=64, H=H, K=K)
    fa = T.compile(ga["inputs"], ga["outputs"], updates=ga["updates"], exclude=("fuse_narrow_grad",))
    gb = C.build_mlp(T, B=B, D=64, H=H, K=K)
    fb = T.compile(gb["inputs"], gb["outputs"], updates=gb["updates"])
    kinds = [getattr(n.op, "display_name", n.op.name) for n in fb.order]
    assert kinds.count("narrow_grad+sgd+db") == 2 and "dot+mul_1msqr" not in kinds
    for _ in range(3):
        ca, cb = fa(x, y)[0], fb(x, y)[0]
        assert abs(ca - cb) <= 1e-5 * abs(ca)
    for pa, pb in zip(ga["params"], gb["params"]):
        a, b = pa.get_value(), pb.get_value()
        assert np.linalg.norm(a - b) <= 1e-5 * max(np.linalg.norm(a), 1e-30), pa.name


@pytest.mark.parametrize("N,K", [(20, 10000), (7, 3000), (300, 257), (64, 10240), (300, 256), (50, 10241), (3, 2)])
def test_wide_row_fusion_softmax_xent(N, K):
    """Vocabulary-sized rows (one 1024-thread CTA per row): softmax +
    cross-entropy forward and gradient, max / argmax outputs, against the
    unfused graph (sums to reassociation, max / argmax bit-exact)."""
    rng = np.random.default_rng(N + K)
    z = T.matrix("z", dtype="float32")
    y = T.matrix("y", dtype="float32")
    m = T.max(z, axis=1)
    e = T.exp(z - T.dimshuffle(m, (0, "x")))
    p = e / T.dimshuffle(T.sum(e, axis=1), (0, "x"))
    cost = -T.sum(y * T.log(p)) / float(N)
    (gz,) = T.grad(cost, [z])
    outs = [cost, gz, m, T.argmax(z, axis=1), T.sum(gz, axis=0)]
    fa = T.compile([z, y], outs, row_fusion=False)
    fb = T.compile([z, y], outs)
    plan_groups = None
    zv = (rng.standard_normal((N, K)) * 3).astype(np.float32)
    zv[0, min(5, K - 1)] = zv[0, max(K - 3, 0)] = 50.0  # a tie at the row maximum
    yv = np.eye(K, dtype=np.float32)[rng.integers(0, K, N)]
    a, b = fa(zv, yv), fb(zv, yv)
    plan_groups = next(iter(fb._plans.values())).row_groups
    from paper_1605_02688_b200.rowfuse import MAX_WIDE
    assert bool(plan_groups and any(g.K == K for g in plan_groups)) == (2 <= K <= MAX_WIDE and N != K)
    assert abs(a[0] - b[0]) <= 1e-5 * abs(a[0])
    np.testing.assert_allclose(b[1], a[1], rtol=1e-5, atol=1e-8)
    np.testing.assert_array_equal(b[2], a[2])
    np.testing.assert_array_equal(b[3], a[3])
    np.testing.assert_allclose(b[4], a[4], rtol=1e-4, atol=1e-7)
    # and against the reference algorithm itself (CPU oracle, same graph)
    cpu = C.CpuFunction(T, [z, y], outs, exclude=("fuse_elemwise",))
    o = cpu(zv, yv)
    assert abs(b[0] - o[0]) <= 1e-5 * abs(o[0])
    np.testing.assert_allclose(b[1], o[1], rtol=1e-5, atol=1e-8)
    np.testing.assert_array_equal(b[2], o[2])
    np.testing.assert_array_equal(b[3], o[3])
    np.testing.assert_allclose(b[4], o[4], rtol=1e-4, atol=1e-7)


@pytest.mark.parametrize("A,B,K", [(20, 20, 10000), (6, 7, 130), (3, 50, 257)])
def test_rank3_row_fusion_softmax_xent(A, B, K):
    """Softmax / cross-entropy over the last axis of an [A, B, K] tensor (the
    stacked per-step logits the loop rewrites move out of an LSTM): the A*B
    rows are one fused row space; results equal the unfused graph."""
    rng = np.random.default_rng(A * B + K)
    z = T.tensor3("z", dtype="float32")
    y = T.tensor3("y", dtype="float32")
    m = T.max(z, axis=2)
    e = T.exp(z - T.dimshuffle(m, (0, 1, "x")))
    p = e / T.dimshuffle(T.sum(e, axis=2), (0, 1, "x"))
    cost = -T.sum(y * T.log(p)) / float(A * B)
    (gz,) = T.grad(cost, [z])
    outs = [cost, gz, m, T.argmax(z, axis=2)]
    fa = T.compile([z, y], outs, row_fusion=False)
    fb = T.compile([z, y], outs)
    zv = (rng.standard_normal((A, B, K)) * 3).astype(np.float32)
    yv = np.eye(K, dtype=np.float32)[rng.integers(0, K, (A, B))]
    a, b = fa(zv, yv), fb(zv, yv)
    groups = next(iter(fb._plans.values())).row_groups
    assert any(g.lead == (A, B) and g.K == K for g in groups)
    assert abs(a[0] - b[0]) <= 1e-5 * abs(a[0])
    np.testing.assert_allclose(b[1], a[1], rtol=1e-5, atol=1e-8)
    np.testing.assert_array_equal(b[2], a[2])
    np.testing.assert_array_equal(b[3], a[3])


def test_mlp_full_size_3xtf32_three_steps_vs_oracle():
    """Config 4 at full size (B=8192, H=4096) with fp32-equivalent tensor-core
    GEMMs: three SGD steps within 1e-5 of the reference algorithm (cost rtol,
    parameter relative L2) -- the precision the reference's sgemm has."""
    B = 8192
    g = C.build_mlp(T, B=B)
    x, y = C.inputs_mlp(B=B)
    step = T.compile(g["inputs"], g["outputs"], updates=g["updates"], gemm_mode="3xtf32")
    gc = C.build_mlp(T, B=B)
    cpu = C.CpuFunction(T, gc["inputs"], gc["outputs"], gc["updates"], exclude=("fuse_elemwise",))
    for _ in range(3):
        c_dev, c_ref = float(step(x, y)[0]), float(cpu(x, y)[0])
        assert abs(c_dev - c_ref) <= 1e-5 * abs(c_ref), (c_dev, c_ref)
    for i, (p, q) in enumerate(zip(g["params"], gc["params"])):
        assert rel(p.get_value(), cpu.value(q)) <= 1e-5, i
