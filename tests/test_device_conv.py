"""2-d convolution trio on the device (im2col -> tensor-core GEMM, col2im
gather) against the REAL reference's outputs (tests/golden/make_conv_golden.py)
and NumPy, plus reshape / shape_of and the implementation-selection rules
(reference ops/conv.py, rewrites/convselect.py)."""
import ctypes
import os
import sys

import numpy as np
import pytest

import paper_1605_02688_b200 as T
from paper_1605_02688_b200.errors import AbstractOpRemaining, ShapeMismatch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, GOLD)
from make_conv_golden import CASES, case_inputs  # noqa: E402


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(np.asarray(b, np.float64)), 1e-30))


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("impl", ["gemm", "reference"])
def test_conv_trio_matches_reference(case, impl):
    g = np.load(os.path.join(GOLD, "ref_conv_goldens.npz"))
    name, dt, xs, fs, st, pd, seed = case
    x, f, _ = case_inputs(dt, xs, fs, seed)
    vx, vf = T.tensor4("x", dtype=dt), T.tensor4("f", dtype=dt)
    y = T.conv2d(vx, vf, stride=st, pad=pd)
    w = T.as_variable(g[f"{name}_w"])
    gx, gf = T.grad(T.sum(y * w), [vx, vf])
    fn = T.compile([vx, vf], [y, gx, gf], conv_impl=impl)
    assert all(n.op.algo == impl for n in fn.order if n.op.name == "conv2d")
    # float64 and exact-fp32 ("reference") are tight; fp32 "gemm" runs TF32 tensor cores
    tol = 1e-12 if dt == "float64" else (1e-6 if impl == "reference" else 3e-3)
    for got, k in zip(fn(x, f), ("y", "gx", "gf")):
        assert got.shape == g[f"{name}_{k}"].shape
        assert _rel(got, g[f"{name}_{k}"]) <= tol, (k, _rel(got, g[f"{name}_{k}"]))


def test_conv_forward_numpy_oracle_and_errors(rng):
    x = rng.standard_normal((3, 4, 11, 9)).astype(np.float32)
    f = rng.standard_normal((6, 4, 3, 3)).astype(np.float32)
    vx, vf = T.tensor4("x", dtype="float32"), T.tensor4("f", dtype="float32")
    (y,) = T.compile([vx, vf], [T.conv2d(vx, vf, stride=(2, 2), pad=(1, 1))], conv_impl="reference")(x, f)
    xp = np.pad(x.astype(np.float64), ((0, 0), (0, 0), (1, 1), (1, 1)))
    want = np.zeros((3, 6, 6, 5))
    for i in range(6):
        for j in range(5):
            win = xp[:, :, 2 * i: 2 * i + 3, 2 * j: 2 * j + 3]
            want[:, :, i, j] = np.einsum("nchw,kchw->nk", win, f.astype(np.float64))
    assert _rel(y, want) <= 1e-6
    # every implementation excluded: refused at compile time (reference rewrites/engine.py:328-340);
    # no selection stage at all: the placeholder fails when it is executed
    with pytest.raises(T.NoImplementationSelected):
        T.compile([vx, vf], [T.conv2d(vx, vf)], conv_impl="none")
    with pytest.raises(AbstractOpRemaining):
        T.compile([vx, vf], [T.conv2d(vx, vf)], preset="none")(x, f)
    with pytest.raises(ShapeMismatch):
        T.compile([vx, vf], [T.conv2d(vx, vf)])(x, rng.standard_normal((6, 5, 3, 3)).astype(np.float32))


def test_reshape_and_shape_of(rng):
    x = T.tensor3("x", dtype="float32")
    r = T.reshape(x, (4, -1))
    s = T.shape_of(x)
    g = T.grad(T.sum(r * r), x)
    fn = T.compile([x], [r, s, g])
    xv = rng.standard_normal((2, 4, 3)).astype(np.float32)
    rv, sv, gv = fn(xv)
    np.testing.assert_array_equal(rv, xv.reshape(4, 6))
    np.testing.assert_array_equal(sv, [2, 4, 3])
    np.testing.assert_array_equal(gv, 2 * xv)
    xt = T.transpose(T.matrix("m", dtype="float32"))
    (tv,) = T.compile([xt.owner.inputs[0]], [T.reshape(xt, (-1,))])(np.arange(6, dtype=np.float32).reshape(2, 3))
    np.testing.assert_array_equal(tv, np.arange(6).reshape(2, 3).T.reshape(-1))


def _conv_ref(x, f, st, pd):
    """Direct-loop cross-correlation (float64) and its two gradients for an
    all-ones upstream weight w: dy = w."""
    N, C, H, W = x.shape
    K, _, kh, kw = f.shape
    xp = np.pad(x, ((0, 0), (0, 0), (pd[0], pd[0]), (pd[1], pd[1])))
    Ho = (H + 2 * pd[0] - kh) // st[0] + 1
    Wo = (W + 2 * pd[1] - kw) // st[1] + 1
    y = np.zeros((N, K, Ho, Wo))
    for i in range(Ho):
        for j in range(Wo):
            win = xp[:, :, i * st[0]: i * st[0] + kh, j * st[1]: j * st[1] + kw]
            y[:, :, i, j] = np.einsum("nchw,kchw->nk", win, f)
    return y


@pytest.mark.parametrize("seed", range(12))
def test_conv_random_shapes_and_gradients(seed):
    """Random NCHW / KCHW shapes, strides and paddings: the forward against
    direct loops, and both gradients against central finite differences of
    the direct-loop forward (float64, exact)."""
    rng = np.random.default_rng(900 + seed)
    N, C, K = (int(v) for v in rng.integers(1, 4, 3))
    kh, kw = (int(v) for v in rng.integers(1, 4, 2))
    st = tuple(int(v) for v in rng.integers(1, 3, 2))
    pd = tuple(int(v) for v in rng.integers(0, 2, 2))
    H = int(rng.integers(kh, kh + 6))
    W = int(rng.integers(kw, kw + 6))
    x = rng.standard_normal((N, C, H, W))
    f = rng.standard_normal((K, C, kh, kw))
    vx, vf = T.tensor4("x"), T.tensor4("f")
    y = T.conv2d(vx, vf, stride=st, pad=pd)
    yr = _conv_ref(x, f, st, pd)
    wv = rng.standard_normal(yr.shape)
    gx, gf = T.grad(T.sum(y * T.as_variable(wv)), [vx, vf])
    got_y, got_gx, got_gf = T.compile([vx, vf], [y, gx, gf])(x, f)
    assert _rel(got_y, yr) <= 1e-12
    # exact gradients of a linear map: <w, conv(x, f)> is linear in x and in f
    eps = 1.0
    gx_ref = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        d = np.zeros_like(x)
        d[idx] = eps
        gx_ref[idx] = (wv * _conv_ref(d, f, st, pd)).sum()
    gf_ref = np.zeros_like(f)
    for idx in np.ndindex(*f.shape):
        d = np.zeros_like(f)
        d[idx] = eps
        gf_ref[idx] = (wv * _conv_ref(x, d, st, pd)).sum()
    assert _rel(got_gx, gx_ref) <= 1e-12
    assert _rel(got_gf, gf_ref) <= 1e-12


def _conv_nhwc_ref(xpad, w, kh, kw):
    """out[(n,p,q), k] = sum_{u,v,c} xpad[n,p+u,q+v,c] w[k,(u,v,c)] in float64, and |.| bound."""
    N, Hp, Wp, C = xpad.shape
    P, Q = Hp - kh + 1, Wp - kw + 1
    X = xpad.astype(np.float64)
    Wt = w.astype(np.float64).reshape(w.shape[0], kh, kw, C)
    out = np.zeros((N, P, Q, w.shape[0]))
    bound = np.zeros_like(out)
    for u in range(kh):
        for v in range(kw):
            patch = X[:, u:u + P, v:v + Q, :]
            out += patch @ Wt[:, u, v, :].T
            bound += np.abs(patch) @ np.abs(Wt[:, u, v, :]).T
    return out.reshape(N * P * Q, -1), bound.reshape(N * P * Q, -1)


@pytest.mark.parametrize("N,Hp,Wp,C,K,kh,kw", [(2, 10, 12, 32, 64, 3, 3), (1, 58, 58, 64, 64, 3, 3),
                                                (3, 9, 130, 32, 40, 3, 3), (2, 20, 7, 96, 300, 5, 5),
                                                (4, 5, 5, 64, 16, 1, 1), (1, 33, 67, 32, 64, 2, 4)])
def test_conv_implicit_gemm_direct(N, Hp, Wp, C, K, kh, kw):
    """tx_conv_implicit through the C ABI: the A tile of every (tap, channel
    block) is a 4-D TMA box of the padded NHWC input (ragged last row block,
    output width up to 128, several output-channel tiles, 1x1 and 5x5 taps);
    TF32 products against float64 within 2^-9 of the |x||w| bound."""
    import torch
    from paper_1605_02688_b200 import native
    if Wp - kw + 1 > 128:
        pytest.skip("output width > 128 is outside the implicit path")
    lib = native.library()
    rng = np.random.default_rng(N * 1000 + C + K)
    xpad = rng.standard_normal((N, Hp, Wp, C)).astype(np.float32)
    w = rng.standard_normal((K, kh * kw * C)).astype(np.float32)
    P, Q = Hp - kh + 1, Wp - kw + 1
    tx, tw = torch.from_numpy(xpad).cuda(), torch.from_numpy(w).cuda()
    to = torch.full((N * P * Q, K), float("nan"), device="cuda")
    mk = native.make_tensor
    win = (ctypes.c_int * 2)(kh, kw)
    lib.check(lib.lib.tx_conv_implicit(mk(tx.data_ptr(), "float32", xpad.shape, (Hp * Wp * C, Wp * C, C, 1)),
                                       mk(tw.data_ptr(), "float32", w.shape, (w.shape[1], 1)),
                                       mk(to.data_ptr(), "float32", (N * P * Q, K), (K, 1)), win, None))
    torch.cuda.synchronize()
    got = to.cpu().numpy()
    want, bound = _conv_nhwc_ref(xpad, w, kh, kw)
    assert np.all(np.abs(got - want) <= 2.0 ** -9 * bound + 1e-5), float(np.nanmax(np.abs(got - want) / (bound + 1e-30)))
    # the same product stored straight into an NCHW output
    t4 = torch.full((N, K, P, Q), float("nan"), device="cuda")
    lib.check(lib.lib.tx_conv_implicit(mk(tx.data_ptr(), "float32", xpad.shape, (Hp * Wp * C, Wp * C, C, 1)),
                                       mk(tw.data_ptr(), "float32", w.shape, (w.shape[1], 1)),
                                       mk(t4.data_ptr(), "float32", (N, K, P, Q), (K * P * Q, P * Q, Q, 1)), win, None))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(t4.cpu().numpy(), got.reshape(N, P, Q, K).transpose(0, 3, 1, 2))


@pytest.mark.parametrize("N,C,H,W,ph,pw", [(2, 64, 7, 9, 1, 1), (1, 40, 5, 130, 0, 2), (3, 3, 4, 4, 2, 0)])
def test_pad_nhwc_direct(N, C, H, W, ph, pw):
    """tx_pad_nhwc: NCHW (here a strided, sliced view) -> zero-padded NHWC in
    one pass, bit-exact against NumPy (channel blocks of 32 with a ragged
    last block, borders zeroed without a memset)."""
    import torch
    from paper_1605_02688_b200 import native
    lib = native.library()
    rng = np.random.default_rng(C + W)
    big = rng.standard_normal((N, C, H, W + 3)).astype(np.float32)
    xs = big[:, :, :, 1:W + 1]
    tb = torch.from_numpy(big).cuda()
    ty = torch.full((N, H + 2 * ph, W + 2 * pw, C), float("nan"), device="cuda")
    mk = native.make_tensor
    tx = mk(tb.data_ptr() + 4, "float32", (N, C, H, W), (C * H * (W + 3), H * (W + 3), W + 3, 1))
    pads = (ctypes.c_int * 2)(ph, pw)
    lib.check(lib.lib.tx_pad_nhwc(tx, mk(ty.data_ptr(), "float32", tuple(ty.shape), tuple(ty.stride())), pads, None))
    torch.cuda.synchronize()
    want = np.zeros((N, H + 2 * ph, W + 2 * pw, C), np.float32)
    want[:, ph:ph + H, pw:pw + W, :] = xs.transpose(0, 2, 3, 1)
    np.testing.assert_array_equal(ty.cpu().numpy(), want)


@pytest.mark.parametrize("shape,pad,ks", [((2, 32, 9, 11), (1, 1), 3), ((3, 64, 12, 7), (2, 1), 5),
                                          ((1, 32, 6, 130), (0, 0), 3), ((2, 96, 5, 5), (0, 0), 1)])
def test_conv_trio_implicit_vs_exact(shape, pad, ks):
    """The stride-1, 32-channel-block layers take the implicit-GEMM forward
    and input gradient (and the weight gradient's patch matrix from the padded
    NHWC buffer): forward and both gradients within TF32 tolerance of the
    exact fp32 CUDA-core lowering (conv_impl="reference")."""
    rng = np.random.default_rng(sum(shape) + ks)
    N, C, H, W = shape
    K = 64 if C > 64 else (32 if ks != 5 else 24)   # K % 32 == 0: the input gradient is implicit too
    x = rng.standard_normal(shape).astype(np.float32)
    f = (rng.standard_normal((K, C, ks, min(ks, 3))) / np.sqrt(C * ks * 3)).astype(np.float32)
    vx, vf = T.tensor4("x", dtype="float32"), T.tensor4("f", dtype="float32")
    y = T.conv2d(vx, vf, stride=(1, 1), pad=pad)
    gf, gx = T.grad(T.sum(y * y), [vf, vx])
    outs = {}
    for impl in ("gemm", "reference"):
        outs[impl] = T.compile([vx, vf], [y, gf, gx], conv_impl=impl)(x, f)
    for a, b in zip(outs["gemm"], outs["reference"]):
        assert a.shape == b.shape
        assert _rel(a, b) <= 3e-3, _rel(a, b)
