"""Per-op parity of the B200 kernels against the reference's golden vectors
and the CPU oracle.  Tolerances:
  - add/sub/mul/div/neg/sqr/sqrt/maximum/second/switch, comparisons, isnan,
    max, argmax (both forms), integer ops: bit-exact;
  - exp/log/log1p/tanh/sigmoid/pow: |d-o| <= 1e-6 + 1e-5|o| (f32), CUDA libm
    vs NumPy SIMD differ by ulps;
  - sum: |d-o| <= 2e-6 * sum|x|;
  - TF32 GEMM: |C-C_o| <= 2^-9 (|A||B|)_ij + 1e-6 (operands rounded to TF32);
    CUDA-core GEMM paths: |C-C_o| <= 1e-5 (|A||B|)_ij + 1e-6.
"""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import texpr_numpy as O
from paper_1605_02688_b200.elemwise import make
from paper_1605_02688_b200.errors import ShapeMismatch

pytestmark = pytest.mark.gpu

EXACT = ("add", "sub", "mul", "div", "neg", "sqr", "sqrt", "maximum", "second", "lt", "gt", "le", "ge", "eq",
         "neq", "isnan")
TRANSC = ("exp", "log", "log1p", "tanh", "sigmoid", "pow")


def close(got, want, rtol, atol):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    nan_g, nan_w = np.isnan(got), np.isnan(want)
    assert np.array_equal(nan_g, nan_w)
    ok = ~nan_w
    inf = np.isinf(want) & ok
    assert np.array_equal(got[inf], want[inf])
    fin = ok & ~inf
    np.testing.assert_allclose(got[fin], want[fin], rtol=rtol, atol=atol)


def exact(got, want):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    if got.dtype.kind == "f":
        assert np.array_equal(np.isnan(got), np.isnan(want))
        m = ~np.isnan(want)
        assert np.array_equal(got[m], want[m])
        # bit-exact includes the sign of zero (== treats -0.0 and +0.0 as equal)
        assert np.array_equal(np.signbit(got[m]), np.signbit(want[m]))
    else:
        assert np.array_equal(got, want)


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_elementwise_kernels(golden, dt):
    a, b, c = golden[f"ew_{dt}_a"], golden[f"ew_{dt}_b"], golden[f"ew_{dt}_c"]
    va, vb, vc = T.vector("a", dtype=dt), T.vector("b", dtype=dt), T.vector("c", dtype="bool")
    tol = (1e-5, 1e-6) if dt == "float32" else (1e-12, 1e-14)
    for k in EXACT + ("pow",):
        if k in ("neg", "sqr", "sqrt", "isnan"):
            got = T.compile([va], make(k, [va]), preset="none")(a)
        else:
            got = T.compile([va, vb], make(k, [va, vb]), preset="none")(a, b)
        want = golden[f"ew_{dt}_{k}"]
        if k in EXACT:
            exact(got, want)
        else:
            close(got, want, *tol)
    for k in TRANSC:
        if k == "pow":
            continue
        got = T.compile([va], make(k, [va]), preset="none")(a)
        close(got, golden[f"ew_{dt}_{k}"], *tol)
    exact(T.compile([vc, va, vb], make("switch", [vc, va, vb]), preset="none")(c, a, b), golden[f"ew_{dt}_switch"])


def test_integer_kernels_and_zero_division(golden):
    a, b = golden["ew_int64_a"], golden["ew_int64_b"]
    va, vb = T.vector("a", dtype="int64"), T.vector("b", dtype="int64")
    for k in ("add", "sub", "mul", "div", "maximum", "lt", "eq"):
        exact(T.compile([va, vb], make(k, [va, vb]), preset="none")(a, b), golden[f"ew_int64_{k}"])
    f = T.compile([va, vb], make("div", [va, vb]), preset="none")
    with pytest.raises(ZeroDivisionError):
        f(a, np.zeros_like(b))


def test_broadcast_composite(golden):
    vX = T.matrix("X", dtype="float32")
    vr = T.vector("r", dtype="float32")
    vcol = T.matrix("col", dtype="float32", broadcastable=(False, True))
    f = T.compile([vX, vr, vcol], T.tanh(vX + vr) * vcol - vr)
    close(f(golden["bc_X"], golden["bc_r"], golden["bc_col"]), golden["bc_out"], 1e-5, 1e-6)


def test_elementwise_rank3_rank4_row_forms(rng):
    """Rank-3/4 iteration spaces that do not collapse to 2-D -- a time-reversed
    view and a [T]-vector broadcast over [T, B, V] (the LSTM loss layer), a
    4-D mix of broadcasts -- take the row-major kernels with per-row
    coordinates (ew_template.cuh TX_ROW_COORDS), vectorised and scalar:
    bit-identical to NumPy float32 arithmetic."""
    Tn, B, V = 5, 6, 36
    X = rng.standard_normal((Tn, B, V)).astype(np.float32)
    Y = rng.standard_normal((Tn, B, V)).astype(np.float32)
    t = rng.standard_normal(Tn).astype(np.float32)
    m = rng.standard_normal((Tn, B)).astype(np.float32)
    vX, vY = T.tensor3("X", dtype="float32"), T.tensor3("Y", dtype="float32")
    vt, vm = T.vector("t", dtype="float32"), T.matrix("m", dtype="float32")
    expr = (vX[::-1] + T.dimshuffle(vt, (0, "x", "x"))) * vY - T.dimshuffle(vm, (0, 1, "x"))
    f = T.compile([vX, vY, vt, vm], expr)
    want = (X[::-1] + t[:, None, None]) * Y - m[:, :, None]
    exact(f(X, Y, t, m), want)
    # odd row length: the scalar row form
    exact(f(X[:, :, :35].copy(), Y[:, :, :35].copy(), t, m), (X[::-1, :, :35] + t[:, None, None]) * Y[:, :, :35] - m[:, :, None])
    # rank 4: [A, B, C, D] with a [A, 1, C, 1] and a [1, B, 1, D] operand
    A4 = rng.standard_normal((3, 4, 5, 8)).astype(np.float32)
    p = rng.standard_normal((3, 5)).astype(np.float32)
    q = rng.standard_normal((4, 8)).astype(np.float32)
    vA = T.tensor4("A", dtype="float32")
    vp, vq = T.matrix("p", dtype="float32"), T.matrix("q", dtype="float32")
    g = T.compile([vA, vp, vq], vA * T.dimshuffle(vp, (0, "x", 1, "x")) + T.dimshuffle(vq, ("x", 0, "x", 1)))
    exact(g(A4, p, q), A4 * p[:, None, :, None] + q[None, :, None, :])


def test_config2_expression_fused(golden):
    r7 = np.random.default_rng(7)
    ins = [r7.standard_normal(40000, dtype=np.float32) for _ in range(4)]
    a, b, c, d = (T.vector(s, dtype="float32") for s in "abcd")
    f = T.compile([a, b, c, d], T.sigmoid(a * b + c) ** 2 - d)
    assert sum(1 for n in f.order if n.op.name == "composite") == 1 and len(f.order) == 1
    close(f(*ins), golden["cfg2_fused"], 1e-5, 1e-6)
    # unaligned / odd length exercises the scalar tail and the non-vector path
    g = f(*[x[1:40000 - 3] for x in ins])
    close(g, golden["cfg2_fused"][1:40000 - 3], 1e-5, 1e-6)


@pytest.mark.parametrize("ax", [(0,), (1,), (0, 1)])
def test_reductions_golden(golden, ax):
    X = golden["red_X"]
    v = T.matrix("R", dtype="float32")
    tag = "".join(map(str, ax))
    f = T.compile([v], [T.sum(v, axis=ax), T.max(v, axis=ax), T.argmax_onehot(v, axis=ax)])
    s, m, oh = f(X)
    exact(m, golden[f"red_max_{tag}"])
    exact(oh, golden[f"red_argmax_onehot_{tag}"])
    want = golden[f"red_sum_{tag}"]
    close(s, want, 0, 2e-6 * float(np.nansum(np.abs(X))))


@pytest.mark.parametrize("ax", [(0, 2), (1,), (0, 1, 2), (2,), (0,)])
def test_reductions_rank3_f64(golden, ax):
    X = golden["red3_X"]
    v = T.tensor3("R3", dtype="float64")
    tag = "".join(map(str, ax))
    s, m, oh = T.compile([v], [T.sum(v, axis=ax), T.max(v, axis=ax), T.argmax_onehot(v, axis=ax)])(X)
    exact(m, golden[f"red3_max_{tag}"])
    exact(oh, golden[f"red3_argmax_onehot_{tag}"])
    close(s, golden[f"red3_sum_{tag}"], 1e-12, 1e-12)


@pytest.mark.parametrize("shape", [(4099, 3001), (3, 70000), (70000, 3), (1, 1), (1, 200000), (33, 600),
                                   (4100, 3000), (1001, 1040)])
def test_reduction_forms(shape, rng):
    """ROW / split-ROW / warp-ROW / COL(+splits) / degenerate shapes."""
    X = rng.standard_normal(shape).astype(np.float32)
    X.flat[rng.integers(0, X.size, 3)] = X.max() + 1  # ties at the max
    v = T.matrix("X", dtype="float32")
    for ax in ((0,), (1,), (0, 1)):
        f = T.compile([v], [T.sum(v, axis=ax), T.max(v, axis=ax), T.argmax(v, axis=ax)])
        s, m, am = f(X)
        exact(m, O.reduce_max(X, ax))
        exact(am, O.argmax_index(X, ax))
        close(s, O.reduce_sum(X, ax), 0, 2e-6 * float(np.abs(X).sum()) + 1e-6)


def test_column_reduction_tma_nan_ties_int(rng):
    """Axis-0 reductions on TMA-addressable matrices (16-byte row pitch): the
    COLTMA form (cp.async.bulk.tensor ring) must stay bit-exact for max /
    argmax with NaNs and ties, including a ragged last tile and strip."""
    X = rng.standard_normal((2051, 1300)).astype(np.float32)
    X[7, 3] = X[900, 3] = 50.0          # tie: first row wins
    X[5, 1299] = np.nan                 # NaN propagates / wins argmax
    X[2050, 1299] = np.nan
    X[2050, 0] = 99.0                   # max in the ragged last row tile
    v = T.matrix("X", dtype="float32")
    s, m, am, oh = T.compile([v], [T.sum(v, axis=0), T.max(v, axis=0), T.argmax(v, axis=0),
                                   T.argmax_onehot(v, axis=0)])(X)
    exact(m, O.reduce_max(X, (0,)))
    exact(am, O.argmax_index(X, (0,)))
    exact(oh, O.argmax_onehot(X, (0,)))
    close(s, O.reduce_sum(X, (0,)), 0, 2e-6 * float(np.nansum(np.abs(X))) + 1e-6)
    Xi = rng.integers(-1000, 1000, (3000, 1024)).astype(np.int32)
    vi = T.matrix("Xi", dtype="int32")
    si, mi = T.compile([vi], [T.sum(vi, axis=0), T.max(vi, axis=0)])(Xi)
    exact(mi, Xi.max(axis=0))
    exact(si, Xi.sum(axis=0, dtype=np.int32))


def test_reduction_strided_views(rng):
    X = rng.standard_normal((300, 500)).astype(np.float32)
    v = T.matrix("X", dtype="float32")
    vt = T.transpose(v)
    f = T.compile([v], [T.sum(vt, axis=0), T.max(vt, axis=1), T.argmax(vt, axis=None)])
    s, m, am = f(X)
    close(s, X.T.sum(axis=0), 1e-5, 1e-5)
    exact(m, O.reduce_max(X.T, (1,)))
    exact(am, O.argmax_index(X.T, (0, 1)))


def test_nan_propagation_max_and_argmax():
    X = np.arange(24, dtype=np.float32).reshape(4, 6)
    X[1, 2] = np.nan
    X[2, 5] = np.nan
    X[2, 1] = np.nan
    v = T.matrix("X", dtype="float32")
    m, am, oh = T.compile([v], [T.max(v, axis=1), T.argmax(v, axis=1), T.argmax_onehot(v, axis=0)])(X)
    exact(m, O.reduce_max(X, (1,)))
    exact(am, O.argmax_index(X, (1,)))
    exact(oh, O.argmax_onehot(X, (0,)))


@pytest.mark.parametrize("shape", [(64, 40000), (3, 1 << 20), (257, 4099)])
def test_row_argmax_ties_nan_inf(shape, rng):
    """Row argmax (axis 1 and all axes) over long rows -- many float4 chunks
    per thread, rows split across CTAs -- with repeated maxima in different
    chunks, all -inf rows, NaNs late in a row: first occurrence, NaN wins
    (bit-exact with NumPy)."""
    R, K = shape
    X = rng.integers(-3, 4, size=shape).astype(np.float32)   # heavy ties
    X[0, :] = -np.inf
    X[1, K // 2] = np.nan
    X[1, K - 1] = np.nan
    if R > 2:
        X[2, K - 2] = 7.0
        X[2, 5] = 7.0
    X = X[:, :]
    v = T.matrix("X", dtype="float32")
    f = T.compile([v], [T.argmax(v, axis=1), T.argmax(v), T.max(v, axis=1)])
    am, aall, m = f(X)
    exact(am, O.argmax_index(X, (1,)))
    exact(aall, O.argmax_index(X, (0, 1)))
    exact(m, O.reduce_max(X, (1,)))
    Y = X[:, 1:]  # rows start misaligned: the scalar path
    am2 = T.compile([v], T.argmax(v, axis=1))(np.ascontiguousarray(Y))
    exact(am2, O.argmax_index(Y, (1,)))


def test_dot_golden(golden):
    A, B, v = golden["dot_A"], golden["dot_B"], golden["dot_v"]
    vA, vB, vv = T.matrix("A", dtype="float32"), T.matrix("B", dtype="float32"), T.vector("v", dtype="float32")
    f = T.compile([vA, vB, vv], [T.dot(vA, vB), T.dot(vA, vv), T.dot(vv, vB), T.dot(vv, vv), T.dot(T.transpose(vA), vA)])
    outs = f(A, B, v)
    for got, key, (x, y) in zip(outs, ("dot_mm", "dot_mv", "dot_vm", "dot_vv", "dot_tn"),
                                ((A, B), (A, v), (v, B), (v, v), (A.T, A))):
        bound = np.abs(x).astype(np.float64) @ np.abs(y).astype(np.float64)
        assert np.all(np.abs(got - golden[key]) <= 1e-5 * bound + 1e-6)


def _gemm_case(M, N, K, ta, tb, mode, rng):
    a = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    b = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    ea = T.transpose(va) if ta else va
    eb = T.transpose(vb) if tb else vb
    f = T.compile([va, vb], T.dot(ea, eb), gemm_mode=mode)
    got = f(a, b)
    A = (a.T if ta else a).astype(np.float64)
    B = (b.T if tb else b).astype(np.float64)
    return got, A @ B, np.abs(A) @ np.abs(B)


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (300, 520, 784), (784, 1024, 1000), (1024, 4096, 128), (352, 160, 96),
                                   (20, 3000, 600), (700, 40, 1200), (20, 300, 8192), (64, 64, 20000),
                                   (129, 65, 33)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_tcgen05_layouts(M, N, K, ta, tb, rng):
    assert _gemm_path(M, N, K, ta, tb, 0) == _expected_path(M, N, K, ta, tb)
    got, want, bound = _gemm_case(M, N, K, ta, tb, "auto", rng)
    err = np.abs(got - want)
    assert np.all(err <= 2.0 ** -9 * bound + 1e-6), float((err / (bound + 1e-30)).max())


def _gemm_path(M, N, K, ta, tb, mode):
    """tx_gemm_path for the layouts _gemm_case builds (aligned dummy pointers)."""
    from paper_1605_02688_b200 import native
    lib = native.library()
    mk = native.make_tensor
    a = mk(256, "float32", (M, K), (1, M) if ta else (K, 1))
    b = mk(256, "float32", (K, N), (1, K) if tb else (N, 1))
    c = mk(256, "float32", (M, N), (N, 1))
    return lib.gemm_path(a, b, c, mode)


def _expected_path(M, N, K, ta, tb):
    """The dispatch rule (tx_gemm.cu choose / gemm_tc_eligible) restated: a
    regression that silently routes eligible products to SIMT fails here."""
    if K <= 16 or N <= 16:
        return 1                       # skinny (outer product / row dot / K reduction)
    if M <= 32 and N * K <= 1 << 21:
        return 1                       # few rows: the SIMT small-M kernel (tx_gemm_simt.cu smallm_kernel)
    lead_a = M if ta else K
    lead_b = K if tb else N
    thin_ok = min(M, N) >= 64 or M * N * K >= (1 << 20)
    if lead_a % 4 == 0 and lead_b % 4 == 0 and thin_ok:
        return 2
    return 1 if M <= 16 else 0         # C^T = B^T A^T makes M <= 16 a skinny N


@pytest.mark.parametrize("M,N,K", [(256, 512, 256), (300, 520, 784), (784, 1024, 1000), (1024, 4096, 128), (352, 160, 96),
                                   (20, 3000, 600), (700, 40, 1200), (20, 300, 8192), (64, 64, 20000),
                                   (8192, 4096, 784), (129, 65, 33), (301, 517, 783)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_3xtf32_layouts(M, N, K, ta, tb, rng):
    """fp32-equivalent tensor-core products (gemm_mode="3xtf32"): every tcgen05
    layout within 2^-20 |A||B| of the exact product, i.e. the
    reference's sgemm precision class, and on the tcgen05 path -- also for
    layouts the TF32 path cannot address (the split re-lays the operands)."""
    assert _gemm_path(M, N, K, ta, tb, 3) == 2
    got, want, bound = _gemm_case(M, N, K, ta, tb, "3xtf32", rng)
    err = np.abs(got - want)
    assert np.all(err <= 2.0 ** -20 * bound + 1e-7), float((err / (bound + 1e-30)).max())


@pytest.mark.parametrize("M,N,K", [(20, 800, 200), (20, 200, 800), (1, 33, 17), (7, 1000, 65), (16, 64, 4096),
                                   (32, 200, 10000), (20, 3000, 600), (31, 129, 257), (17, 20, 100000)])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_gemm_small_m(M, N, K, ta, tb, rng):
    """M <= 32 (an unrolled scan's recurrent products): the SIMT small-M
    kernel, every operand layout (N-major, K-major and strided B; both A
    layouts), the cluster split of K (up to 8 CTAs summed through distributed
    shared memory) and ragged column strips -- exact fp32 FMAs."""
    assert _gemm_path(M, N, K, ta, tb, 0) == 1
    got, want, bound = _gemm_case(M, N, K, ta, tb, "auto", rng)
    assert np.all(np.abs(got - want) <= 1e-5 * bound + 1e-6), float((np.abs(got - want) / (bound + 1e-30)).max())


def test_gemm_small_m_strided_and_epilogues(rng):
    """Strided (non-unit) operand views and every fused epilogue kind on the
    small-M path, against the unfused graph (bit-exact: the same product
    followed by the same IEEE round-to-nearest epilogue arithmetic)."""
    M, N, K = 20, 200, 150
    x = rng.standard_normal((M, 2 * K)).astype(np.float32)
    w = rng.standard_normal((K, 3 * N)).astype(np.float32)
    g = rng.standard_normal((M, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    vx, vw = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32")
    vg, vb = T.matrix("g", dtype="float32"), T.vector("b", dtype="float32")
    z = T.dot(vx[:, ::2], vw[:, ::3])
    outs = [z, T.tanh(z + vb), z * vg, z * (1.0 - vg * vg), (vg + z) + vb]
    fused = T.compile([vx, vw, vg, vb], outs)(x, w, g, bias)
    plain = T.compile([vx, vw, vg, vb], outs, exclude=("fuse_gemm_epilogue",))(x, w, g, bias)
    want = x[:, ::2].astype(np.float64) @ w[:, ::3].astype(np.float64)
    bound = np.abs(x[:, ::2]).astype(np.float64) @ np.abs(w[:, ::3]).astype(np.float64)
    assert np.all(np.abs(fused[0] - want) <= 1e-5 * bound + 1e-6)
    for a, b in zip(fused, plain):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("M,N,K", [(8192, 10, 4096), (600, 10, 784), (8192, 4096, 10), (784, 10, 600),
                                   (4096, 10, 8192), (5, 300, 77), (7, 9, 11)])
def test_gemm_skinny_and_simt_exactish(M, N, K, rng):
    for ta in (False, True):
        got, want, bound = _gemm_case(M, N, K, ta, False, "auto", rng)
        assert np.all(np.abs(got - want) <= 1e-5 * bound + 1e-6)


def test_gemm_simt_mode_and_f64(rng):
    got, want, bound = _gemm_case(200, 300, 150, True, False, "simt", rng)
    assert np.all(np.abs(got - want) <= 1e-5 * bound + 1e-6)
    a = rng.standard_normal((70, 50))
    b = rng.standard_normal((50, 90))
    va, vb = T.matrix("a"), T.matrix("b")
    np.testing.assert_allclose(T.compile([va, vb], T.dot(va, vb))(a, b), a @ b, rtol=1e-12, atol=1e-12)


def test_dot_shape_mismatch_raises():
    va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    f = T.compile([va, vb], T.dot(va, vb))
    with pytest.raises(ShapeMismatch):
        f(np.zeros((3, 4), np.float32), np.zeros((5, 6), np.float32))


def _narrow_case(B, H, k, rng, sgd=False, pad_h=0, dtype=np.float32, mode=0, rtol=1e-5):
    """tx_narrow_grad through the C ABI vs the oracle's three separate ops."""
    import ctypes

    import torch

    from paper_1605_02688_b200 import native
    lib = native.device_library(0)
    dz = (rng.standard_normal((B, k)) * 1e-2).astype(dtype)
    W = (rng.standard_normal((H, k)) * 0.05).astype(dtype)
    h = np.tanh(rng.standard_normal((B, H))).astype(dtype)
    want_dh = O.dot(dz, W.T) * (1 - h * h)
    want_gw = O.dot(h.T, dz)
    want_db = want_dh.astype(np.float64).sum(0)
    tdev = {}
    # h (and dh) optionally as row-padded views: ragged row pitch -> fallback path
    hp = np.zeros((B, H + pad_h), dtype)
    hp[:, :H] = h
    tdev["dz"], tdev["W"], tdev["h"] = (torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (dz, W, hp))
    tdev["dh"] = torch.zeros((B, H + pad_h), dtype=getattr(torch, np.dtype(dtype).name), device="cuda")
    tdev["gw"] = tdev["W"] if sgd else torch.zeros((H, k), dtype=tdev["W"].dtype, device="cuda")
    tdev["db"] = torch.zeros(H, dtype=tdev["W"].dtype, device="cuda")
    dt = np.dtype(dtype).name
    mk = native.make_tensor
    tdz = mk(tdev["dz"].data_ptr(), dt, (B, k), (k, 1))
    twt = mk(tdev["W"].data_ptr(), dt, (k, H), (1, k))
    th = mk(tdev["h"].data_ptr(), dt, (B, H), (H + pad_h, 1))
    tdh = mk(tdev["dh"].data_ptr(), dt, (B, H), (H + pad_h, 1))
    tgw = mk(tdev["gw"].data_ptr(), dt, (H, k), (k, 1))
    tdb = mk(tdev["db"].data_ptr(), dt, (H,), (1,))
    epi = native.TxEpilogue()
    lr = 0.25
    if sgd:
        epi.kind = native.EPI_SGD
        epi.aux = mk(tdev["W"].data_ptr(), dt, (H, k), (k, 1))
        epi.alpha = lr
    wsb = lib.narrow_grad_workspace(tdz, twt, th, tdh, tgw, tdb, mode)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    lib.check(lib.lib.tx_narrow_grad(tdz, twt, th, tdh, tgw, ctypes.byref(epi), tdb, mode,
                                     ctypes.c_void_p(ws.data_ptr()), wsb, None))
    torch.cuda.synchronize()
    dh = tdev["dh"].cpu().numpy()[:, :H]
    scale = O.dot(np.abs(dz), np.abs(W.T)) + 1e-30
    # products are exact-fp32 FMAs (CUDA cores): reassociation-level error only
    assert np.all(np.abs(dh - want_dh) <= rtol * scale + 1e-7)
    gw = tdev["gw"].cpu().numpy()
    gscale = O.dot(np.abs(h.T), np.abs(dz)) + 1e-30
    if sgd:
        want_w = W - np.float32(lr) * want_gw
        assert np.all(np.abs(gw - want_w) <= lr * (rtol * gscale) + 1e-6 * np.abs(W) + 1e-7)
    else:
        assert np.all(np.abs(gw - want_gw) <= rtol * gscale + 1e-7)
    db = tdev["db"].cpu().numpy()
    dscale = np.abs(O.dot(np.abs(dz), np.abs(W.T))).sum(0) if rtol > 1e-5 else np.abs(want_dh).sum(0)
    assert np.all(np.abs(db - want_db) <= max(rtol, 2e-6) * dscale + 1e-7)


@pytest.mark.parametrize("B,H,k", [(8192, 4096, 10), (1, 4, 1), (37, 1028, 16), (4100, 2052, 3), (40, 36, 7)])
def test_narrow_grad_fused(B, H, k, rng):
    _narrow_case(B, H, k, rng)


def test_narrow_grad_sgd_in_place_and_fallbacks(rng):
    _narrow_case(2048, 512, 10, rng, sgd=True)                  # fused, SGD epilogue writing over W
    _narrow_case(300, 130, 10, rng, pad_h=2)                    # unaligned rows -> tx_gemm x2 + tx_reduce
    _narrow_case(300, 128, 17, rng, mode=1)                      # k > 16 -> fallback (exact-fp32 GEMM mode)
    _narrow_case(96, 64, 5, rng, sgd=True, dtype=np.float64)   # float64 -> fallback
    # wide k on the tensor cores: db from the dh GEMM's epilogue column sums (TF32 products)
    _narrow_case(1000, 256, 128, rng, sgd=True, rtol=2.0 ** -9)
    _narrow_case(70, 96, 64, rng, rtol=2.0 ** -9)


@pytest.mark.parametrize("M", [1, 4, 16, 37])
def test_dot_bias_epilogues_short_m(M, rng):
    """dot + row bias (and tanh) with few rows: the M <= 16 products run
    transposed on the skinny kernels, where the bias runs along the other
    axis (regression: every column used bias[0])."""
    x = rng.standard_normal((M, 32)).astype(np.float32)
    W = rng.standard_normal((32, 50)).astype(np.float32)
    b = rng.standard_normal(50).astype(np.float32)
    vx, vw, vb = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32"), T.vector("b", dtype="float32")
    want = x.astype(np.float64) @ W + b
    f = T.compile([vx, vw, vb], T.dot(vx, vw) + vb)
    assert "dot+bias" in [getattr(n.op, "display_name", n.op.name) for n in f.order]
    np.testing.assert_allclose(f(x, W, b), want, rtol=1e-5, atol=1e-5)
    # the forward layer with its tanh-gradient factor: dot+bias_tanh_dual
    h = T.tanh(T.dot(vx, vw) + vb)
    g = T.compile([vx, vw, vb], [h, 1.0 - T.sqr(h)])
    hv, gv = g(x, W, b)
    np.testing.assert_allclose(hv, np.tanh(want), rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(gv, 1 - np.tanh(want) ** 2, rtol=1e-5, atol=1e-5)


def test_dot_bias_strided_and_unaligned_bias(rng):
    """The tensor-core epilogue with a bias that is a strided or unaligned
    view (every other element of a vector, or a vector starting one element
    into its buffer)."""
    x = rng.standard_normal((256, 128)).astype(np.float32)
    W = rng.standard_normal((128, 192)).astype(np.float32)
    bb = rng.standard_normal(2 * 192 + 1).astype(np.float32)
    vx, vw, vb = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32"), T.vector("bb", dtype="float32")
    for sl, bview in ((slice(0, 2 * 192, 2), bb[: 2 * 192: 2]), (slice(1, 193, None), bb[1:193])):
        f = T.compile([vx, vw, vb], T.dot(vx, vw) + T.subtensor(vb, (sl,)))
        assert "dot+bias" in [getattr(n.op, "display_name", n.op.name) for n in f.order]
        got = f(x, W, bb)
        want = x.astype(np.float64) @ W + bview
        bound = np.abs(x).astype(np.float64) @ np.abs(W)
        assert np.all(np.abs(got - want) <= 2.0 ** -9 * bound + 1e-5)
    # a bias of the wrong length fails like the unfused add would
    from paper_1605_02688_b200.errors import ShapeMismatch
    f = T.compile([vx, vw, vb], T.dot(vx, vw) + vb)
    with pytest.raises(ShapeMismatch):
        f(x, W, bb)


def test_reductions_over_empty_extents():
    """Zero-size inputs: an empty result launches nothing, a sum over an
    empty axis is 0, max / argmax over one raise (NumPy's ValueError in the
    reference) -- the planner used to divide by the empty extent (SIGFPE)."""
    from paper_1605_02688_b200.errors import TexprError
    x = T.tensor3("x")
    for shape in ((2, 33, 0), (5, 0, 33), (0, 0, 1)):
        xv = np.zeros(shape)
        s0, s1 = T.compile([x], [T.sum(x, axis=0), T.sum(x, axis=1)])(xv)
        np.testing.assert_array_equal(s0, xv.sum(0))
        np.testing.assert_array_equal(s1, xv.sum(1))
        if 0 in (shape[1],):
            with pytest.raises(Exception):
                T.compile([x], T.max(x, axis=1))(xv)
        else:
            np.testing.assert_array_equal(T.compile([x], T.max(x, axis=1))(xv), xv.max(1))


def test_empty_operands_everywhere():
    """Zero-size operands through every kernel family: fused elementwise,
    GEMMs with an empty M / N / K (K = 0 gives zeros), a softmax region over
    zero rows, a loop over zero steps."""
    x, w = T.matrix("x"), T.matrix("w")
    e = T.tanh(x * 2.0 + 1.0) - x
    m = T.max(x, axis=1)
    p = T.exp(x - T.dimshuffle(m, (0, "x")))
    sm = p / T.dimshuffle(T.sum(p, axis=1), (0, "x"))
    f = T.compile([x, w], [e, T.dot(x, w), sm])
    for xs, ws in (((0, 5), (5, 3)), ((4, 0), (0, 3)), ((4, 5), (5, 0))):
        xv, wv = np.ones(xs), np.ones(ws)
        if xs[1] == 0:
            got = T.compile([x, w], [e, T.dot(x, w)])(xv, wv)
            want = [np.tanh(xv * 2 + 1) - xv, xv @ wv]
        else:
            got = f(xv, wv)
            ev = np.exp(xv - xv.max(1, keepdims=True)) if xv.size else xv
            want = [np.tanh(xv * 2 + 1) - xv, xv @ wv, ev / ev.sum(1, keepdims=True) if xv.size else ev]
        for g, wnt in zip(got, want):
            assert g.shape == wnt.shape
            np.testing.assert_allclose(g, wnt)
    xs = T.matrix("xs")
    h0 = T.vector("h0")
    (hist,), (final,) = T.scan(lambda x_t, h: [T.tanh(x_t + h)], sequences=[xs], initial_states=[h0])
    hv, fv = T.compile([xs, h0], [hist, final])(np.zeros((0, 3)), np.ones(3))
    assert hv.shape == (0, 3)
    np.testing.assert_array_equal(fv, np.ones(3))


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_signed_zeros_bit_exact(dt):
    """maximum / switch / second / neg / sub and the max reduction on +-0.0
    (with ties, NaN and infinities around them) reproduce NumPy's sign of
    zero (the reference's kernels, ops/elemwise.py:91-113, ops/reductions.py:126)."""
    vals = np.array([0.0, -0.0, -0.0, 0.0, 1.0, -1.0, np.nan, np.inf, -np.inf, -0.0], dtype=dt)
    a = np.array(np.meshgrid(vals, vals)[0].ravel(), dtype=dt)
    b = np.array(np.meshgrid(vals, vals)[1].ravel(), dtype=dt)
    c = (np.arange(a.size) % 3 == 0)
    va, vb, vc = T.vector("a", dtype=dt), T.vector("b", dtype=dt), T.vector("c", dtype="bool")
    for k in ("maximum", "sub", "add", "mul"):
        exact(T.compile([va, vb], make(k, [va, vb]), preset="none")(a, b), O.elemwise(k, [a, b]))
    exact(T.compile([va], make("neg", [va]), preset="none")(a), O.elemwise("neg", [a]))
    exact(T.compile([vc, va, vb], make("switch", [vc, va, vb]), preset="none")(c, a, b),
          O.elemwise("switch", [c, a, b]))
    exact(T.compile([va, vb], make("second", [va, vb]), preset="none")(a, b), O.elemwise("second", [a, b]))
    m = T.matrix("m", dtype=dt)
    Z = np.array([[0.0, -0.0, 0.0], [-0.0, 0.0, -0.0], [-0.0, -0.0, -0.0], [0.0, 0.0, -0.0]] * 70, dtype=dt)
    for ax in ((0,), (1,), None):
        got = T.compile([m], T.max(m, axis=ax))(Z)
        exact(got, O.reduce_max(Z, (0, 1) if ax is None else ax))


@pytest.mark.parametrize("K", [3, 40, 700])
def test_signed_zero_max_inside_row_fusion(K):
    """The row max of a fused softmax region (rowfuse.py, warp- and
    block-per-row forms) on rows whose maximum is +-0: the sign of the last
    zero -- NumPy's sequential semantics (v = maximum(v, x), ties keep the
    later operand).  NumPy's own SIMD reduce over >= 16 contiguous elements
    combines lanes in an order that depends on the host CPU's vector width,
    so the reference's sign of a zero maximum is itself host-dependent there;
    np.maximum.accumulate is the sequential definition."""
    rng = np.random.default_rng(K)
    z = -np.abs(rng.standard_normal((64, K))).astype(np.float32) - 1.0
    for r in range(64):
        cols = rng.choice(K, size=min(K, 1 + r % 3), replace=False)
        z[r, cols] = np.where(rng.random(cols.size) < 0.5, np.float32(0.0), np.float32(-0.0))
    v = T.matrix("z", dtype="float32")
    m = T.max(v, axis=1)
    e = T.exp(v - T.dimshuffle(m, (0, "x")))
    p = e / T.dimshuffle(T.sum(e, axis=1), (0, "x"))
    f = T.compile([v], [m, p])
    got_m, got_p = f(z)
    assert next(iter(f._plans.values())).row_groups, "expected a fused row region"
    exact(got_m, np.maximum.accumulate(z, axis=1)[:, -1])
    np.testing.assert_allclose(got_p, T.compile([v], [p], row_fusion=False)(z)[0], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("M,N,K", [(8, 64, 32), (20, 800, 200), (20, 2400, 600), (300, 520, 784)])
def test_dot_add_aux_bias_epilogue_bit_exact(M, N, K, rng):
    """x.W + g + b (a recurrent pre-activation with its input projection g):
    fused into the GEMM epilogue as b + (g + acc) -- the same two IEEE adds
    as the unfused composite, so the result is bit-identical on every path
    (transposed skinny M <= 16, thin tcgen05 tiles, the regular tiles)."""
    x = rng.standard_normal((M, K)).astype(np.float32)
    W = rng.standard_normal((K, N)).astype(np.float32)
    g = rng.standard_normal((M, N)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32)
    vx, vw = T.matrix("x", dtype="float32"), T.matrix("w", dtype="float32")
    vg, vb = T.matrix("g", dtype="float32"), T.vector("b", dtype="float32")
    expr = (vg + T.dot(vx, vw)) + vb
    f = T.compile([vx, vw, vg, vb], expr)
    assert "dot+add_aux_bias" in [getattr(n.op, "display_name", n.op.name) for n in f.order]
    u = T.compile([vx, vw, vg, vb], expr, exclude=("fuse_gemm_epilogue",))
    assert "dot+add_aux_bias" not in [getattr(n.op, "display_name", n.op.name) for n in u.order]
    np.testing.assert_array_equal(f(x, W, g, b), u(x, W, g, b))


@pytest.mark.parametrize("M,N,K", [(784, 3072, 512), (1000, 3072, 256), (784, 4096, 1024)])
def test_gemm_a_panel_multicast(M, N, K, rng):
    """Single-CTA one-wave products with an MN-major A (xᵀ·dz, the MLP's
    weight gradient) run with the A panel multicast across 4-CTA clusters
    along N (ragged last M tile included), plain and with the fused SGD
    epilogue: within the TF32 bound of the float64 product.  (75-148 output
    tiles: one wave and no split-K, the multicast condition.)"""
    a = rng.standard_normal((K, M)).astype(np.float32)     # A = aᵀ (MN-major)
    b = rng.standard_normal((K, N)).astype(np.float32)
    w = rng.standard_normal((M, N)).astype(np.float32)
    va, vb = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    got = T.compile([va, vb], T.dot(T.transpose(va), vb))(a, b)
    A, B = a.T.astype(np.float64), b.astype(np.float64)
    want, bound = A @ B, np.abs(A) @ np.abs(B)
    assert np.all(np.abs(got - want) <= 2.0 ** -9 * bound + 1e-6)
    W = T.shared(w.copy(), name="W")
    f = T.compile([va, vb], [], updates=[(W, W - 0.5 * T.dot(T.transpose(va), vb))])
    f(a, b)
    upd = W.get_value()
    assert np.all(np.abs(upd - (w - 0.5 * want)) <= 0.5 * 2.0 ** -9 * bound + 1e-5)
