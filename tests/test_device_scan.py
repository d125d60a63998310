"""Symbolic loops on the device, mirroring the reference's tests/test_scan.py:
forward semantics, BPTT gradients and R-operator against explicitly unrolled
graphs (built with subtensor/join, the reference's own oracle construction,
tests/helpers.py:15-35) and against plain NumPy loops."""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from paper_1605_02688_b200.errors import LengthMismatch, MissingNonSequence, TypeMismatch
from paper_1605_02688_b200.ops import dimshuffle, join, subtensor
from paper_1605_02688_b200.scan import LAST, scan

pytestmark = pytest.mark.gpu


def expand0(v):
    return dimshuffle(v, ("x",) + tuple(range(v.type.ndim)))


def unroll(fn, sequences, initial_states, non_sequences, length):
    states = list(initial_states)
    collected = []
    for t in range(length):
        xs = [subtensor(s, (t,)) for s in sequences]
        outs = fn(*xs, *states, *non_sequences)
        outs = [outs] if isinstance(outs, T.Variable) else list(outs)
        if not collected:
            collected = [[] for _ in outs]
        for i, o in enumerate(outs):
            collected[i].append(o)
        states = outs[: len(initial_states)]
    return [join(0, *[expand0(o) for o in h]) for h in collected], states


def rel_err(a, b, floor=1e-12):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def run(inputs, outputs, values, **kw):
    return T.compile(inputs, outputs, **kw)(*values)


def test_cumulative_sum():
    xs, s0 = T.vector("xs"), T.scalar("s0")
    (hist,), (final,) = scan(lambda x, s: s + x, sequences=[xs], initial_states=[s0])
    h, f = run([xs, s0], [hist, final], [np.array([1.0, 2.0, 3.0]), np.array(0.0)])
    np.testing.assert_array_equal(h, [1.0, 3.0, 6.0])
    assert float(f) == 6.0


def test_zero_steps_returns_initial_state():
    s0 = T.vector("s0")
    (hist,), (final,) = scan(lambda s: s * 2.0, initial_states=[s0], n_steps=0)
    h, f = run([s0], [hist, final], [np.array([7.0, 8.0])])
    assert h.shape == (0, 2)
    np.testing.assert_array_equal(f, [7.0, 8.0])


def test_sequences_length_mismatch():
    a, b = T.vector("a"), T.vector("b")
    (h,), _ = scan(lambda x, y, s: s + x * y, sequences=[a, b], initial_states=[T.as_variable(0.0)])
    with pytest.raises(LengthMismatch):
        run([a, b], [h], [np.arange(3.0), np.arange(4.0)])


def test_n_steps_input_value_keys_the_plan():
    a = T.vector("a")
    n = T.make_input(T.tensor_type("int64", 0), "n")
    (h,), _ = scan(lambda x, s: s + x, sequences=[a], initial_states=[T.as_variable(0.0)], n_steps=n)
    f = T.compile([a, n], [h])
    np.testing.assert_array_equal(f(np.arange(3.0), np.array(3, np.int64))[0], [0.0, 1.0, 3.0])
    with pytest.raises(LengthMismatch):
        f(np.arange(3.0), np.array(5, np.int64))
    s0 = T.scalar("s0")
    (h2,), (f2,) = scan(lambda s: s * 2.0, initial_states=[s0], n_steps=n)
    g = T.compile([s0, n], [h2, f2])
    for steps in (4, 2, 0):
        hv, fv = g(np.array(1.5), np.array(steps, np.int64))
        np.testing.assert_array_equal(hv, 1.5 * 2.0 ** np.arange(1, steps + 1))
        assert float(fv) == 1.5 * 2.0 ** steps


def test_construction_errors():
    s0 = T.scalar("s0")
    with pytest.raises(LengthMismatch):
        scan(lambda s: s + 1.0, initial_states=[s0])
    w = T.scalar("w")
    with pytest.raises(MissingNonSequence):
        scan(lambda s: s * w, initial_states=[s0], n_steps=3, strict=True)
    with pytest.raises(TypeMismatch):
        scan(lambda s: T.fill(T.as_variable(np.zeros(3)), s) + 1.0, initial_states=[s0], n_steps=2)


def test_nonstrict_captures_become_invariants():
    s0, w = T.scalar("s0"), T.scalar("w")
    (hist,), _ = scan(lambda s: s * w, initial_states=[s0], n_steps=4)
    assert hist.owner.op.n_nonseqs == 1
    (h,) = run([s0, w], [hist], [np.array(1.0), np.array(3.0)])
    np.testing.assert_array_equal(h, [3.0, 9.0, 27.0, 81.0])


def _rnn(dtype="float64"):
    xs, h0 = T.matrix("xs", dtype=dtype), T.vector("h0", dtype=dtype)
    w, u = T.matrix("w", dtype=dtype), T.matrix("u", dtype=dtype)

    def step(x_t, h_prev, w_, u_):
        return T.tanh(T.dot(w_, h_prev) + T.dot(u_, x_t))
    return step, xs, h0, w, u


def _rnn_point(rng, length=5, size=3, dtype=np.float64):
    return [(rng.standard_normal((length, size)) * 0.5).astype(dtype), (rng.standard_normal(size) * 0.5).astype(dtype),
            (rng.standard_normal((size, size)) * 0.4).astype(dtype), (rng.standard_normal((size, size)) * 0.4).astype(dtype)]


def test_rnn_matches_unrolled_and_numpy(rng):
    step, xs, h0, w, u = _rnn()
    (hist,), (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    (uhist,), ustates = unroll(step, [xs], [h0], [w, u], length=5)
    pt = _rnn_point(rng)
    gh, gf, uh, uf = run([xs, h0, w, u], [hist, final, uhist, ustates[0]], pt)
    h, ref = pt[1], []
    for t in range(5):
        h = np.tanh(pt[2] @ h + pt[3] @ pt[0][t])
        ref.append(h)
    assert rel_err(gh, uh) <= 1e-12 and rel_err(gf, uf) <= 1e-12
    assert rel_err(gh, np.array(ref)) <= 1e-12


def test_rnn_gradients_match_unrolled(rng):
    step, xs, h0, w, u = _rnn()
    _, (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    _, ustates = unroll(step, [xs], [h0], [w, u], length=5)
    wrt = [xs, h0, w, u]
    grads = T.grad(T.sum(T.sqr(final)), wrt)
    ugrads = T.grad(T.sum(T.sqr(ustates[0])), wrt)
    pt = _rnn_point(rng)
    got = run(wrt, grads, pt)
    want = run(wrt, ugrads, pt)
    for g, wv, name in zip(got, want, "xs h0 w u".split()):
        assert rel_err(g, wv) <= 1e-10, name


def test_final_cumsum_gradient_is_ones(rng):
    xs, s0 = T.vector("xs"), T.scalar("s0")
    _, (final,) = scan(lambda x, s: s + x, sequences=[xs], initial_states=[s0])
    (gv,) = run([xs, s0], [T.grad(final, xs)], [rng.standard_normal(6), np.array(0.0)])
    np.testing.assert_array_equal(gv, np.ones(6))


def test_rop_cumsum_is_cumsum_of_direction(rng):
    xs, s0 = T.vector("xs"), T.scalar("s0")
    (hist,), _ = scan(lambda x, s: s + x, sequences=[xs], initial_states=[s0])
    v, v0 = T.vector("v"), T.scalar("v0")
    r = T.rop([hist], [xs, s0], [v, v0])[0]
    d = rng.standard_normal(4)
    (rv,) = run([xs, s0, v, v0], [r], [rng.standard_normal(4), np.array(0.0), d, np.array(0.0)])
    np.testing.assert_allclose(rv, np.cumsum(d), rtol=1e-12)


def test_rnn_rop_matches_unrolled(rng):
    step, xs, h0, w, u = _rnn()
    _, (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    _, ustates = unroll(step, [xs], [h0], [w, u], length=3)
    dirs = [T.matrix("dxs"), T.vector("dh0"), T.matrix("dw"), T.matrix("du")]
    r = T.rop([final], [xs, h0, w, u], dirs)[0]
    ur = T.rop([ustates[0]], [xs, h0, w, u], dirs)[0]
    pt = _rnn_point(rng, length=3)
    dv = [rng.standard_normal(p.shape) for p in pt]
    got, want = run([xs, h0, w, u] + dirs, [r, ur], pt + dv)
    assert rel_err(got, want) <= 1e-10


def test_unrolled_grad_equivalence_with_extras(rng):
    for seed in range(3):
        r = np.random.default_rng(seed + 90)
        length = int(r.integers(1, 6))
        xs, h0, w = T.vector("xs"), T.scalar("h0"), T.scalar("w")

        def step(x, s, w_):
            return T.tanh(s * w_ + x) + T.sigmoid(x * s)
        (hist,), (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w])
        (uhist,), ustates = unroll(step, [xs], [h0], [w], length=length)
        grads = T.grad(T.sum(hist * hist) + final, [xs, h0, w])
        ugrads = T.grad(T.sum(uhist * uhist) + ustates[0], [xs, h0, w])
        vals = [r.standard_normal(length) * 0.6, np.array(r.standard_normal() * 0.3), np.array(0.7)]
        for g, wv in zip(run([xs, h0, w], grads, vals), run([xs, h0, w], ugrads, vals)):
            assert rel_err(g, wv) <= 1e-10


def test_nested_loop_forward_and_grad(rng):
    xs, a0 = T.vector("xs"), T.scalar("a0")

    def outer_step(x_t, acc):
        _, (inner_final,) = scan(lambda s, x: T.tanh(s + x), initial_states=[acc], non_sequences=[x_t], n_steps=3)
        return acc * 0.5 + inner_final
    (hist,), (final,) = scan(outer_step, sequences=[xs], initial_states=[a0])
    xv, a = rng.standard_normal(4) * 0.5, 0.2
    expect, acc = [], a
    for t in range(4):
        s = acc
        for _ in range(3):
            s = np.tanh(s + xv[t])
        acc = acc * 0.5 + s
        expect.append(acc)
    gx = T.grad(final, [xs, a0])
    h, f, g0, g1 = run([xs, a0], [hist, final] + gx, [xv, np.array(a)])
    assert rel_err(h, np.array(expect)) <= 1e-12
    # central differences of the NumPy loop
    def fwd(xv_, a_):
        acc_ = a_
        for t in range(len(xv_)):
            s = acc_
            for _ in range(3):
                s = np.tanh(s + xv_[t])
            acc_ = acc_ * 0.5 + s
        return acc_
    eps = 1e-6
    fd = [(fwd(xv + eps * np.eye(4)[i], a) - fwd(xv - eps * np.eye(4)[i], a)) / (2 * eps) for i in range(4)]
    assert rel_err(g0, fd) <= 1e-6
    assert abs(float(g1) - (fwd(xv, a + eps) - fwd(xv, a - eps)) / (2 * eps)) <= 1e-6


def test_last_retention_keeps_one_step(rng):
    xs, s0 = T.vector("xs"), T.scalar("s0")
    (hist,), (final,) = scan(lambda x, s: s * 0.5 + x, sequences=[xs], initial_states=[s0])
    op = hist.owner.op.with_retention((LAST,))
    outs = T.apply(op, list(hist.owner.inputs))
    xv = rng.standard_normal(7)
    h, f = run([xs, s0], [outs[0], outs[1]], [xv, np.array(0.25)])
    s = 0.25
    for x in xv:
        s = s * 0.5 + x
    assert h.shape == (1,) and abs(float(h[0]) - s) <= 1e-12 and abs(float(f) - s) <= 1e-12


def test_float32_lstm_cell_on_tensor_cores(rng):
    """A float32 gated recurrence whose body GEMMs run on the tcgen05 path
    (batch 128, hidden 256): forward and BPTT gradients vs the unrolled graph
    (same kernels, so agreement is to fp32 reassociation)."""
    B, D, H, L = 128, 64, 256, 6
    xs = T.tensor3("xs", dtype="float32")
    h0, c0 = T.matrix("h0", dtype="float32"), T.matrix("c0", dtype="float32")
    Wx, Wh = T.matrix("Wx", dtype="float32"), T.matrix("Wh", dtype="float32")

    def cell(x, h, c, wx, wh):
        z = T.dot(x, wx) + T.dot(h, wh)
        i, f, o, g = (subtensor(z, (slice(None), slice(k * H, (k + 1) * H))) for k in range(4))
        c2 = T.sigmoid(f) * c + T.sigmoid(i) * T.tanh(g)
        return T.sigmoid(o) * T.tanh(c2), c2
    (hh, _), (hf, cf) = scan(cell, sequences=[xs], initial_states=[h0, c0], non_sequences=[Wx, Wh])
    _, (uh, uc) = unroll(cell, [xs], [h0, c0], [Wx, Wh], length=L)
    cost, ucost = T.sum(T.sqr(hf)), T.sum(T.sqr(uh))
    gw = T.grad(cost, [Wx, Wh])
    ugw = T.grad(ucost, [Wx, Wh])
    vals = [rng.standard_normal((L, B, D)).astype(np.float32), (rng.standard_normal((B, H)) * 0.1).astype(np.float32),
            np.zeros((B, H), np.float32), (rng.standard_normal((D, 4 * H)) * 0.1).astype(np.float32),
            (rng.standard_normal((H, 4 * H)) * 0.05).astype(np.float32)]
    ins = [xs, h0, c0, Wx, Wh]
    got = run(ins, [hf, cost] + gw, vals)
    want = run(ins, [uh, ucost] + ugw, vals)
    for g, wv in zip(got, want):
        assert np.linalg.norm(g - wv) <= 1e-4 * np.linalg.norm(wv)


def test_scan_graph_document_round_trip(rng):
    step, xs, h0, w, u = _rnn()
    (hist,), (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    ins, outs, _, _ = T.load_graph(T.dump_graph([xs, h0, w, u], [hist, final]))
    pt = _rnn_point(rng)
    a = run([xs, h0, w, u], [hist, final], pt)
    b = run(ins, outs, pt)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


# -- pinned to the REAL reference (tests/golden/make_scan_golden.py) ----------

def _ref_gold():
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_scan_goldens.npz"))


def test_rnn_matches_reference_goldens():
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from make_scan_golden import rnn_point
    g = _ref_gold()
    step, xs, h0, w, u = _rnn()
    dirs = [T.matrix("dxs"), T.vector("dh0"), T.matrix("dw"), T.matrix("du")]
    (hist,), (final,) = scan(step, sequences=[xs], initial_states=[h0], non_sequences=[w, u])
    cost = T.sum(T.sqr(final)) + T.sum(hist * 0.5)
    grads = T.grad(cost, [xs, h0, w, u])
    jv = T.rop([final], [xs, h0, w, u], dirs)[0]
    got = run([xs, h0, w, u] + dirs, [hist, final] + grads + [jv], rnn_point())
    for v, k in zip(got, ["rnn_hist", "rnn_final", "rnn_gxs", "rnn_gh0", "rnn_gw", "rnn_gu", "rnn_rop"]):
        assert rel_err(v, g[k]) <= 1e-11, k


def test_nested_and_last_step_match_reference_goldens():
    g = _ref_gold()
    xv, a0 = T.vector("xv"), T.scalar("a0")

    def outer_step(x_t, acc):
        _, (inner_final,) = scan(lambda s, x: T.tanh(s + x), initial_states=[acc], non_sequences=[x_t], n_steps=3)
        return acc * 0.5 + inner_final
    (nh,), (nf,) = scan(outer_step, sequences=[xv], initial_states=[a0])
    gn = T.grad(nf, [xv, a0])
    r = np.random.default_rng(11)
    got = run([xv, a0], [nh, nf] + gn, [r.standard_normal(6) * 0.5, np.array(0.2)])
    for v, k in zip(got, ["nest_hist", "nest_final", "nest_gx", "nest_ga"]):
        assert rel_err(v, g[k]) <= 1e-11, k
    ys = T.vector("ys")
    (lh,), _ = scan(lambda x, s: s * 0.9 + T.tanh(x), sequences=[ys], initial_states=[T.as_variable(0.0)])
    f = T.compile([ys], [lh[-1] * 2.0])
    assert any(n.op.name == "scan" and n.op.retention == ("last",) for n in f.order)
    (v,) = f(np.random.default_rng(13).standard_normal(40))
    assert rel_err(v, g["last_out"]) <= 1e-12


LOOP_REWRITES = ("loop_pushout_sequences", "loop_pushout_accumulators", "loop_pushout_outputs",
                 "loop_drop_unused_outputs")


def test_sequence_pushout_moves_work_out_of_both_loops():
    """The loop rewrites: the BPTT loop's recomputed forward step and
    cross-entropy, the forward loop's input projection and its per-step
    softmax / cross-entropy, and the weight-gradient accumulators run once
    over stacked sequences / histories outside the loops (seq_dot / seq_gram
    GEMMs); results equal the loops without the rewrites, and a saved
    function stays portable."""
    from paper_1605_02688_b200.scan import ScanOp, SeqDot, SeqGram
    from tools.lstm_bench import build
    import torch

    step_a, host = build(T, 32, 6, B=4, V=50, exclude=LOOP_REWRITES)
    step_b, _ = build(T, 32, 6, B=4, V=50)
    ins = [torch.from_numpy(v).cuda() for v in host]
    n_seqdot = sum(isinstance(n.op, SeqDot) for n in step_b.order)
    assert n_seqdot >= 3 and not any(isinstance(n.op, (SeqDot, SeqGram)) for n in step_a.order)
    assert sum(isinstance(n.op, SeqGram) for n in step_b.order) >= 2
    loops = [n.op for n in step_b.order if isinstance(n.op, ScanOp)]
    assert all(op.n_states == 2 for op in loops)  # only the recurrences (h, c / their adjoints) stay carried
    for _ in range(2):
        ca = float(step_a.call_device(*ins, sync=True)[0].item())
    del step_a
    step_c = T.load(step_b.save())
    for _ in range(2):
        cb = float(step_b.call_device(*ins, sync=True)[0].item())
    assert abs(ca - cb) <= 1e-4 * abs(ca)
    cc = float(step_c.call_device(*ins, sync=True)[0].item())
    assert np.isfinite(cc)
