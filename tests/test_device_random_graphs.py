"""Semantic preservation on random graphs (the reference's property test
``test_rewrites.py:306-319`` runs 40 random graphs through its rewrites at
rel 1e-10): here 80 (f64) + 40 (f32) seeded random expression graphs — elementwise ops with
row/column broadcasting, sum/max/argmax over either axis, dot, dimshuffle,
softmax / log-softmax / cross-entropy-shaped row regions —
are compiled for the device (fast_run: fusion, GEMM epilogues, row fusion)
and compared with the reference algorithm on the oracle kernels
(``oracle.configs.CpuFunction``: same preset minus the device-only GEMM
rewrites, NumPy per node).

Tolerances: float64 |d - o| <= 1e-9 * max|o| (CUDA libm vs NumPy differ by
an ulp, amplified by at most a few cancellations), float32 4e-5 * max|o|
(3e-3 at the large shape, whose products run on TF32 tensor cores);
NaN / inf positions must agree exactly and argmax indices bit-exactly.
"""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C
from paper_1605_02688_b200.elemwise import make

pytestmark = pytest.mark.gpu

R, Cc = 37, 53
UNARY = ("neg", "tanh", "sigmoid", "sqr", "exp")
BINARY = ("add", "sub", "mul", "maximum")


def _random_graph(seed, dt, R=R, Cc=Cc):
    rng = np.random.default_rng(seed)
    x = T.matrix("x", dtype=dt)
    y = T.matrix("y", dtype=dt)
    w = T.matrix("w", dtype=dt)         # [C, C] for dot
    v = T.vector("v", dtype=dt)         # [C] row-broadcast operand
    inputs = [x, y, w, v]
    mats, vecs_c, vecs_r = [x, y], [v], []

    def pick(pool):
        return pool[int(rng.integers(len(pool)))]
    for _ in range(int(rng.integers(6, 14))):
        r = rng.random()
        if r < 0.22:
            k = UNARY[int(rng.integers(len(UNARY)))]
            a = pick(mats)
            if k == "exp":
                a = T.tanh(a)            # keep exp's argument bounded
            mats.append(make(k, [a]))
        elif r < 0.55:
            k = BINARY[int(rng.integers(len(BINARY)))]
            a = pick(mats)
            s = rng.random()
            if s < 0.5:
                b = pick(mats)
            elif s < 0.75 and vecs_c:
                b = pick(vecs_c)                          # [C] broadcast over rows
            elif vecs_r:
                b = T.dimshuffle(pick(vecs_r), (0, "x"))  # [R,1] broadcast over columns
            else:
                b = pick(mats)
            mats.append(make(k, [a, b] if rng.random() < 0.5 else [b, a]))
        elif r < 0.75:
            a = pick(mats)
            ax = int(rng.integers(2))
            red = T.sum if rng.random() < 0.6 else T.max
            (vecs_c if ax == 0 else vecs_r).append(red(a, axis=ax))
        elif r < 0.82:
            mats.append(T.dot(pick(mats), w))
        elif r < 0.9:
            # softmax-shaped row regions (what row fusion groups): max, exp,
            # row sums, division, log, one-hot of the row argmax
            a = pick(mats)
            m = T.max(a, axis=1)
            e = T.exp(a - T.dimshuffle(m, (0, "x")))
            p = e / T.dimshuffle(T.sum(e, axis=1), (0, "x"))
            k = int(rng.integers(3))
            if k == 0:
                mats.append(p)
            elif k == 1:
                vecs_r.append(-T.sum(T.tanh(pick(mats)) * T.log(p), axis=1))
            else:
                mats.append(T.argmax_onehot(a, axis=1) * p + T.log(p))
        else:
            if vecs_r:
                mats.append(pick(mats) * T.dimshuffle(T.tanh(pick(vecs_r)), (0, "x")))
            else:
                mats.append(T.tanh(pick(mats)) + pick(mats))
    outs = [mats[-1]]
    if vecs_c:
        outs.append(vecs_c[-1])
    if vecs_r:
        outs.append(vecs_r[-1])
    if rng.random() < 0.5:
        outs.append(T.argmax(mats[-1], axis=int(rng.integers(2))))
    outs.append(T.sum(mats[int(rng.integers(len(mats)))]))
    vals = [rng.standard_normal((R, Cc)), rng.standard_normal((R, Cc)),
            rng.standard_normal((Cc, Cc)) / np.sqrt(Cc), rng.standard_normal(Cc)]
    return inputs, outs, [a.astype(dt) for a in vals]


def _check(got, want, rel):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape and got.dtype == want.dtype
    if want.dtype.kind in "iu":
        np.testing.assert_array_equal(got, want)
        return
    assert np.array_equal(np.isnan(got), np.isnan(want))
    inf = np.isinf(want)
    assert np.array_equal(got[inf], want[inf])
    fin = np.isfinite(want)
    if fin.any():
        scale = np.abs(want[fin]).max()
        assert np.abs(got[fin] - want[fin]).max() <= rel * max(scale, 1e-300)


@pytest.mark.parametrize("dt,rel,shape,n", [("float64", 1e-9, (R, Cc), 80), ("float32", 4e-5, (R, Cc), 40),
                                             # large enough for the tcgen05 GEMM (TF32), COLTMA and 2-D kernels
                                             ("float32", 3e-3, (300, 520), 24)])
def test_random_graphs_match_reference_algorithm(dt, rel, shape, n):
    for seed in range(n):
        inputs, outs, vals = _random_graph(1000 + seed, dt, *shape)
        dev = T.compile(inputs, outs)
        ref = C.CpuFunction(T, inputs, outs)
        got = dev(*vals)
        want = ref(*vals)
        for g, w in zip(got, want):
            _check(g, w, rel)


def _random_view_graph(seed, dt, n=48):
    """Square operands so shape-preserving views mix freely: transposes,
    reversed rows / columns (negative strides), comparisons and switch."""
    from paper_1605_02688_b200.ops import flip0, subtensor
    rng = np.random.default_rng(seed)
    x, y, w = T.matrix("x", dtype=dt), T.matrix("y", dtype=dt), T.matrix("w", dtype=dt)
    pool = [x, y, w]

    def pick():
        return pool[int(rng.integers(len(pool)))]
    for _ in range(int(rng.integers(5, 12))):
        r = rng.random()
        if r < 0.2:
            pool.append(T.dimshuffle(pick(), (1, 0)))
        elif r < 0.32:
            pool.append(flip0(pick()))
        elif r < 0.42:
            pool.append(subtensor(pick(), (slice(None), slice(None, None, -1))))
        elif r < 0.62:
            k = ("add", "mul", "sub", "maximum")[int(rng.integers(4))]
            pool.append(make(k, [pick(), pick()]))
        elif r < 0.72:
            a, b = pick(), pick()
            pool.append(make("switch", [make("gt", [a, b]), a, make("neg", [b])]))
        elif r < 0.86:
            pool.append(T.dot(pick(), pick()))
        else:
            pool.append(T.tanh(pick()) * T.dimshuffle(T.sum(pick(), axis=int(rng.integers(2))), (0, "x")))
    outs = [pool[-1], T.sum(pool[int(rng.integers(3, len(pool)))], axis=0), T.max(pool[-1], axis=1)]
    vals = [(rng.standard_normal((n, n)) / np.sqrt(n)).astype(dt) for _ in range(3)]
    return [x, y, w], outs, vals


@pytest.mark.parametrize("dt,rel", [("float64", 1e-9), ("float32", 4e-5)])
def test_random_view_graphs_match_reference_algorithm(dt, rel):
    for seed in range(40):
        inputs, outs, vals = _random_view_graph(5000 + seed, dt)
        got = T.compile(inputs, outs, gemm_mode="simt" if dt == "float32" else "auto")(*vals)
        want = C.CpuFunction(T, inputs, outs)(*vals)
        for g, w in zip(got, want):
            _check(g, w, rel)


def _random_int_graph(seed, dt, R=29, Cc=41):
    """Integer expressions (bit-exact): add / sub / mul / maximum, floor
    division by a non-zero divisor, comparisons into switch, row / column
    sums and maxima, argmax."""
    rng = np.random.default_rng(seed)
    x, y, v = T.matrix("x", dtype=dt), T.matrix("y", dtype=dt), T.vector("v", dtype=dt)
    mats, vecs = [x, y], [v]

    def pick(pool):
        return pool[int(rng.integers(len(pool)))]
    for _ in range(int(rng.integers(5, 11))):
        r = rng.random()
        if r < 0.4:
            k = ("add", "sub", "mul", "maximum")[int(rng.integers(4))]
            b = pick(mats) if rng.random() < 0.7 else pick(vecs)
            mats.append(make(k, [pick(mats), b]))
        elif r < 0.55:
            d = x if rng.random() < 0.5 else y   # small divisors: d*d + 1 cannot wrap to 0
            mats.append(make("div", [pick(mats), make("add", [make("mul", [d, d]), T.as_variable(np.asarray(1, dtype=dt))])]))
        elif r < 0.7:
            a, b = pick(mats), pick(mats)
            mats.append(make("switch", [make("le", [a, b]), a, make("neg", [b])]))
        elif r < 0.85:
            vecs.append((T.sum if rng.random() < 0.5 else T.max)(pick(mats), axis=0))
        else:
            mats.append(pick(mats) + T.dimshuffle(T.max(pick(mats), axis=1), (0, "x")))
    outs = [mats[-1], vecs[-1], T.argmax(mats[-1], axis=int(rng.integers(2))), T.sum(mats[-1])]
    vals = [rng.integers(-9, 10, (R, Cc)).astype(dt), rng.integers(-9, 10, (R, Cc)).astype(dt),
            rng.integers(-9, 10, Cc).astype(dt)]
    return [x, y, v], outs, vals


@pytest.mark.parametrize("dt", ["int32", "int64"])
def test_random_integer_graphs_bit_exact(dt):
    for seed in range(30):
        inputs, outs, vals = _random_int_graph(7000 + seed, dt)
        got = T.compile(inputs, outs)(*vals)
        want = C.CpuFunction(T, inputs, outs)(*vals)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(np.asarray(g), np.asarray(w))


def test_random_graphs_survive_save_and_load():
    """A compiled random graph saved to a TXFN container and loaded back
    computes the same values (portable form: device-only nodes expanded)."""
    for seed in range(10):
        inputs, outs, vals = _random_graph(1000 + seed, "float64")
        f = T.compile(inputs, outs)
        g = T.load(f.save())
        for a, b in zip(f(*vals), g(*vals)):
            a, b = np.asarray(a), np.asarray(b)
            assert a.shape == b.shape
            assert np.allclose(a, b, rtol=1e-12, atol=1e-12, equal_nan=True)


def test_random_update_graphs_match_reference_algorithm():
    """Shared variables updated from random expressions of each other and of
    the inputs (swaps, views of other shared values, in-place candidates,
    outputs that read the old values), three calls, against the reference
    algorithm's write-back-after-the-step semantics (runtime.py:415-421)."""
    for seed in range(25):
        rng = np.random.default_rng(8000 + seed)
        n = 24
        init = [rng.standard_normal((n, n)), rng.standard_normal((n, n)), rng.standard_normal(n)]

        def build(vals):
            A = T.shared(vals[0].copy(), name="A")
            Bm = T.shared(vals[1].copy(), name="B")
            v = T.shared(vals[2].copy(), name="v")
            x = T.matrix("x")
            pool = [A, Bm, x, T.dimshuffle(A, (1, 0)), Bm * 0.5]
            r = np.random.default_rng(9000 + seed)

            def pick():
                return pool[int(r.integers(len(pool)))]
            for _ in range(int(r.integers(2, 6))):
                k = r.random()
                if k < 0.4:
                    pool.append(pick() + pick())
                elif k < 0.7:
                    pool.append(T.tanh(pick()) * 0.9)
                else:
                    pool.append(T.dot(pick(), pick()) * 0.1)
            choices = [pool[int(r.integers(len(pool)))] for _ in range(2)]
            ups = [(A, choices[0]), (Bm, A if r.random() < 0.4 else choices[1]),
                   (v, v + T.sum(pool[-1], axis=0) * 0.01)]
            outs = [T.sum(pool[-1]), A + 0.0]
            return [x], outs, ups, (A, Bm, v)
        xv = rng.standard_normal((n, n))
        ins, outs, ups, sh_dev = build(init)
        f = T.compile(ins, outs, updates=ups)
        ins2, outs2, ups2, sh_ref = build(init)
        ref = C.CpuFunction(T, ins2, outs2, ups2)
        for _ in range(3):
            got, want = f(xv), ref(xv)
            for g, w in zip(got, want):
                _check(g, w, 1e-9)
        for s_dev, (s_ref, _) in zip(sh_dev, ups2):
            _check(s_dev.get_value(), ref.value(s_ref), 1e-9)


def _random_edge_graph(seed):
    """Rank-3 operands with broadcastable axes, ragged and empty extents,
    reductions over axis pairs, outputs that are inputs or views of them."""
    rng = np.random.default_rng(seed)
    a, b, c = (int(v) for v in rng.choice([0, 2, 5, 33], 3))  # extent 1 only where declared broadcastable
    x = T.tensor3("x")
    y = T.tensor3("y", broadcastable=(False, True, False))       # [a, 1, c]
    v = T.vector("v")                                             # [c]
    pool = [x, y, v]

    def pick():
        return pool[int(rng.integers(len(pool)))]
    for _ in range(int(rng.integers(3, 8))):
        r = rng.random()
        if r < 0.35:
            k = ("add", "mul", "sub", "maximum")[int(rng.integers(4))]
            pool.append(make(k, [pick(), pick()]))
        elif r < 0.5:
            pool.append(T.tanh(pick()))
        elif r < 0.7:
            src = pick()
            if src.type.ndim == 3:
                ax = [(0,), (1,), (2,), (0, 2), (1, 2), (0, 1, 2)][int(rng.integers(6))]
                red = T.sum if rng.random() < 0.6 else T.max
                pool.append(red(src, axis=ax) if len(ax) < 3 else red(src))
        elif r < 0.85:
            src = pick()
            if src.type.ndim == 3:
                pool.append(T.dimshuffle(src, (2, 0, 1)))
        else:
            pool.append(make("second", [pick(), T.as_variable(np.asarray(1.5))]))
    outs = [pool[-1], x, T.dimshuffle(y, (0, 2, 1)), pool[int(rng.integers(len(pool)))]]
    vals = [rng.standard_normal((a, b, c)), rng.standard_normal((a, 1, c)), rng.standard_normal(c)]
    return [x, y, v], outs, vals


def test_random_edge_graphs_match_reference_algorithm():
    """Broadcastable and empty axes, axis-pair reductions, outputs aliasing
    inputs: the device agrees with the reference algorithm or both raise
    (max over an empty axis is an error in both)."""
    for seed in range(60):
        inputs, outs, vals = _random_edge_graph(11000 + seed)
        try:
            want = C.CpuFunction(T, inputs, outs)(*vals)
        except (ValueError, Exception) as exc:  # noqa: B014 (the reference raises on empty max)
            with pytest.raises(Exception):
                T.compile(inputs, outs)(*vals)
            continue
        got = T.compile(inputs, outs)(*vals)
        for g, w in zip(got, want):
            _check(g, w, 1e-9)


def test_random_graphs_under_the_nan_guard():
    """With the NaN guard on, finite random graphs give the unguarded values
    (to reassociation: a guarded step runs without row fusion); a NaN planted
    in an input is reported before anything is returned."""
    from paper_1605_02688_b200.diagnostics import NanGuardConfig
    from paper_1605_02688_b200.errors import NanDetected
    for seed in range(15):
        inputs, outs, vals = _random_graph(1000 + seed, "float64")
        plain = T.compile(inputs, outs)(*vals)
        guarded = T.compile(inputs, outs, nan_guard=NanGuardConfig(big_threshold=None))
        for a, b in zip(plain, guarded(*vals)):
            _check(b, a, 1e-12)
        bad = [v.copy() for v in vals]
        bad[0][3, 4] = np.nan
        with pytest.raises(NanDetected):
            guarded(*bad)


def test_random_lazy_conditionals():
    """ifelse over two random same-typed branches: equals the chosen branch
    compiled alone, for both conditions, and the untaken branch's nodes never
    run (the reference's lazy walk, runtime.py:448-499)."""
    for seed in range(12):
        ins_a, outs_a, vals = _random_graph(1000 + seed, "float64")
        x, y, w, v = ins_a
        # the second branch: another random graph re-expressed over the same inputs
        ins_b, outs_b, _ = _random_graph(2000 + seed, "float64")
        from paper_1605_02688_b200.graph import clone_outputs
        outs_b, _ = clone_outputs(outs_b, dict(zip(ins_b, ins_a)))
        c = T.scalar("c", dtype="int64")
        lazy = T.ifelse(c, outs_a[0], outs_b[0])
        f = T.compile([c] + ins_a, lazy)
        want_a = T.compile(ins_a, outs_a[0])(*vals)
        want_b = T.compile(ins_a, outs_b[0])(*vals)
        _check(f(np.int64(1), *vals), want_a, 1e-12)
        _check(f(np.int64(0), *vals), want_b, 1e-12)
        ran = {nid for nid, k in f.profile.node_calls.items() if k}
        assert ran, "the lazy walk recorded no node calls"


def test_random_graphs_with_changing_shapes():
    """One compiled function called with different row counts in turn (a
    step plan per shape, cached and re-used out of order) agrees with the
    reference algorithm every time."""
    for seed in range(12):
        inputs, outs, _ = _random_graph(1000 + seed, "float64")
        f = T.compile(inputs, outs)
        ref = C.CpuFunction(T, inputs, outs)
        rng = np.random.default_rng(seed)
        for R_ in (37, 5, 64, 37, 5, 1):
            vals = [rng.standard_normal((R_, Cc)), rng.standard_normal((R_, Cc)),
                    rng.standard_normal((Cc, Cc)) / np.sqrt(Cc), rng.standard_normal(Cc)]
            try:
                want = ref(*vals)
            except Exception:
                with pytest.raises(Exception):
                    f(*vals)
                continue
            for g, w in zip(f(*vals), want):
                _check(g, w, 1e-9)


@pytest.mark.slow
def test_random_elementwise_graphs_through_the_host_pipeline():
    """Host-array calls large enough for the chunked H2D / kernel / D2H
    pipeline (stream.py) on random element-wise graphs (ragged length, two
    outputs): identical to the one-shot device call, and to the reference
    algorithm."""
    import torch
    n = (17 << 20) + 12345
    for seed in range(4):
        rng = np.random.default_rng(12000 + seed)
        a, b, c = (T.vector(nm, dtype="float32") for nm in "abc")
        pool = [a, b, c]
        for _ in range(int(rng.integers(3, 8))):
            k = ("add", "mul", "sub", "maximum", "tanh", "sigmoid")[int(rng.integers(6))]
            args = [pool[int(rng.integers(len(pool)))] for _ in range(1 if k in ("tanh", "sigmoid") else 2)]
            pool.append(make(k, args))
        outs = [pool[-1], pool[-2]]
        f = T.compile([a, b, c], outs)
        vals = [rng.standard_normal(n).astype(np.float32) for _ in range(3)]
        host = f(*vals)
        dev = [t.cpu().numpy() for t in f.call_device(*[torch.from_numpy(v).cuda() for v in vals], sync=True)]
        for h, d in zip(host, dev):
            np.testing.assert_array_equal(h, d)
        idx = rng.integers(0, n, 4096)
        want = C.CpuFunction(T, [a, b, c], outs)(*[v[idx] for v in vals])
        for h, w in zip(host, want):
            _check(h[idx], w, 1e-5)


def test_random_graph_gradients_match_directional_differences():
    """grad() of a random scalar cost (the reference's gradient rules,
    autodiff.py / ops/*.py grad) executed on the device agrees with a central
    difference of the device function along a random direction (float64)."""
    for seed in range(15):
        inputs, outs, vals = _random_graph(1000 + seed, "float64")
        rng = np.random.default_rng(seed)
        cost = T.sum(T.tanh(outs[0]) * T.as_variable(rng.standard_normal(vals[0].shape)))
        floats = [v for v in inputs]
        grads = T.grad(cost, floats, disconnected="zero")
        fg = T.compile(inputs, grads)
        fc = T.compile(inputs, cost)
        g = fg(*vals)
        d = [rng.standard_normal(v.shape) for v in vals]
        h = 1e-6
        plus = float(fc(*[v + h * dv for v, dv in zip(vals, d)]))
        minus = float(fc(*[v - h * dv for v, dv in zip(vals, d)]))
        fd = (plus - minus) / (2 * h)
        an = sum(float((np.asarray(gi) * dv).sum()) for gi, dv in zip(g, d))
        assert abs(fd - an) <= 1e-5 * max(1.0, abs(an)), (seed, fd, an)
