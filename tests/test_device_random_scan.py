"""Random recurrences: a loop on the device vs the same body unrolled.

Seeded random recurrent cells (one or two carried states, optional per-step
extra output, tanh / sigmoid / products / row-broadcast biases, dot with
loop-invariant weights, loop lengths 1..6) are built twice: through ``scan``
(compiled for the device: the body compiled once and unrolled into the
captured step, the loop rewrites, BPTT as a reversed loop) and as the
explicitly unrolled graph evaluated by the reference algorithm on the oracle
kernels (``oracle.configs.CpuFunction``) — the reference's own loop test
strategy (``tests/helpers.py:16-39`` unroll oracle).  Forward values and the
gradients w.r.t. the sequence, the initial states and the weights are
compared in float64 (|d - o| <= 1e-9 * max|o|) and float32 (2e-4 * max|o| with
exact-fp32 GEMMs, 3e-3 with TF32 tensor cores).
"""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C

pytestmark = pytest.mark.gpu

B, D = 5, 7


def _cell(rng):
    two = bool(rng.random() < 0.5)
    extra = bool(rng.random() < 0.6)
    act = [T.tanh, T.sigmoid][int(rng.integers(2))]
    mix = int(rng.integers(3))

    def body(x, *rest):
        if two:
            h, c, W, U, b = rest
        else:
            h, W, U, b = rest
            c = None
        z = T.dot(x, W) + T.dot(h, U) + b
        if mix == 0:
            hn = act(z)
        elif mix == 1:
            hn = act(z) * T.tanh(h) + 0.5 * h
        else:
            hn = T.tanh(z - T.dimshuffle(T.max(z, axis=1), (0, "x")))
        outs = [hn]
        if two:
            cn = T.sigmoid(z) * c + T.tanh(hn)
            outs.append(cn)
        if extra:
            outs.append(T.sum(hn * hn, axis=1))
        return outs
    return two, extra, body


def _case(seed, dt="float64", B=B, D=D):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(1, 7))
    two, extra, body = _cell(rng)
    xs = T.tensor3("xs", dtype=dt)
    h0 = T.matrix("h0", dtype=dt)
    c0 = T.matrix("c0", dtype=dt)
    W, U, b = T.matrix("W", dtype=dt), T.matrix("U", dtype=dt), T.vector("b", dtype=dt)
    inits = [h0, c0] if two else [h0]
    inv = [W, U, b]
    outs, finals = T.scan(body, sequences=[xs], initial_states=inits, non_sequences=inv)
    cost = T.sum(T.sqr(finals[0])) + T.sum(outs[0]) + (T.sum(outs[-1]) if extra else 0.0)
    wrt = [xs] + inits + inv
    g_loop = T.grad(cost, wrt, disconnected="zero")
    # the same recurrence, unrolled
    states = list(inits)
    hs, ex = [], []
    for t in range(L):
        r = body(xs[t], *states, *inv)
        states = r[: len(inits)]
        hs.append(states[0])
        if extra:
            ex.append(r[-1])
    cost_u = T.sum(T.sqr(states[0])) + sum(T.sum(h) for h in hs) + (sum(T.sum(e) for e in ex) if extra else 0.0)
    g_unrolled = T.grad(cost_u, wrt, disconnected="zero")
    ins = [xs] + inits + inv
    vals = [rng.standard_normal((L, B, D)), rng.standard_normal((B, D)) * 0.5]
    if two:
        vals.append(rng.standard_normal((B, D)) * 0.5)
    vals += [rng.standard_normal((D, D)) / np.sqrt(D), rng.standard_normal((D, D)) / np.sqrt(D),
             rng.standard_normal(D) * 0.1]
    return ins, [cost] + g_loop, [cost_u] + g_unrolled, [v.astype(dt) for v in vals]


def _close(got, want, rel=1e-9):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    scale = max(np.abs(want).max(), 1e-300) if want.size else 1.0
    assert np.abs(got - want).max() <= rel * scale if want.size else True


# float32: exact-fp32 GEMMs ("simt") at 2e-4; with the default TF32 tensor
# cores the [96 x 24] x [24 x 96] weight-gradient products round their
# operands to TF32 (~2^-11 relative), hence 3e-3
@pytest.mark.parametrize("dt,b,d,rel,n,mode", [("float64", B, D, 1e-9, 30, "auto"),
                                               ("float32", 24, 96, 2e-4, 12, "simt"),
                                               ("float32", 24, 96, 3e-3, 12, "auto")])
def test_random_loops_match_unrolled_reference(dt, b, d, rel, n, mode):
    for seed in range(n):
        ins, loop_outs, unrolled_outs, vals = _case(300 + seed, dt, b, d)
        dev = T.compile(ins, loop_outs, gemm_mode=mode)(*vals)
        ref = C.CpuFunction(T, ins, unrolled_outs)(*vals)
        for k, (g, w) in enumerate(zip(dev, ref)):
            try:
                _close(g, w, rel)
            except AssertionError:
                raise AssertionError(f"seed {300 + seed}: output {k} differs") from None


def test_random_loops_forward_mode_matches_unrolled():
    """R-operator (forward mode) through random loops -- the primal+tangent
    loop of scan.py -- equals the R-operator of the unrolled graph."""
    for seed in range(15):
        rng = np.random.default_rng(600 + seed)
        L = int(rng.integers(1, 6))
        two, extra, body = _cell(rng)
        xs = T.tensor3("xs")
        h0, c0 = T.matrix("h0"), T.matrix("c0")
        W, U, b = T.matrix("W"), T.matrix("U"), T.vector("b")
        inits = [h0, c0] if two else [h0]
        inv = [W, U, b]
        outs, finals = T.scan(body, sequences=[xs], initial_states=inits, non_sequences=inv)
        states = list(inits)
        for t in range(L):
            states = body(xs[t], *states, *inv)[: len(inits)]
        dW, dxs = T.matrix("dW"), T.tensor3("dxs")
        r_loop = T.rop([finals[0]], [W, xs], [dW, dxs])[0]
        r_unr = T.rop([states[0]], [W, xs], [dW, dxs])[0]
        ins = [xs] + inits + inv + [dW, dxs]
        vals = [rng.standard_normal((L, B, D)), rng.standard_normal((B, D)) * 0.5]
        if two:
            vals.append(rng.standard_normal((B, D)) * 0.5)
        vals += [rng.standard_normal((D, D)) / np.sqrt(D), rng.standard_normal((D, D)) / np.sqrt(D),
                 rng.standard_normal(D) * 0.1, rng.standard_normal((D, D)), rng.standard_normal((L, B, D))]
        got = T.compile(ins, r_loop)(*vals)
        want = C.CpuFunction(T, ins, r_unr)(*vals)
        _close(got, want)
