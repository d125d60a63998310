"""Loop construction on the host (no GPU): role/type checks, the BPTT and
R-operator graphs, CSE of the re-applied forward loop, serialization of loop
nodes (reference tests/test_scan.py construction cases)."""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from paper_1605_02688_b200.errors import LengthMismatch, MissingNonSequence, TypeMismatch
from paper_1605_02688_b200.scan import ScanOp, scan


def test_roles_types_and_errors():
    xs, s0, w = T.matrix("xs"), T.vector("s0"), T.scalar("w")
    (hist, ex), (final,) = scan(lambda x, s, w_: [s + x * w_, T.sum(x)], sequences=[xs], initial_states=[s0],
                                non_sequences=[w])
    op = hist.owner.op
    assert isinstance(op, ScanOp) and (op.n_seqs, op.n_states, op.n_nonseqs, op.n_extras) == (1, 1, 1, 1)
    assert hist.type.broadcastable == (False, False) and ex.type.ndim == 1 and final.type == s0.type
    with pytest.raises(LengthMismatch):
        scan(lambda s: s + 1.0, initial_states=[s0])
    with pytest.raises(MissingNonSequence):
        scan(lambda s: s * w, initial_states=[s0], n_steps=3, strict=True)
    with pytest.raises(TypeMismatch):
        scan(lambda x, s: s, sequences=[T.scalar("bad")], initial_states=[s0])


def test_grad_and_rop_graphs_build_and_merge():
    xs, h0, W = T.matrix("xs"), T.vector("h0"), T.matrix("W")
    (hist,), (final,) = scan(lambda x, h, w: T.tanh(T.dot(w, h) + x), sequences=[xs], initial_states=[h0],
                             non_sequences=[W])
    gx, gh, gw = T.grad(T.sum(T.sqr(final)) + T.sum(hist), [xs, h0, W])
    assert gx.type == xs.type and gh.type == h0.type and gw.type == W.type
    f = T.compile([xs, h0, W], [final, gx, gh, gw])
    loops = [n for n in f.order if isinstance(n.op, ScanOp)]
    assert len(loops) == 2  # forward (re-applied inside the gradient, merged by CSE) + reversed
    dirs = [T.matrix("dx"), T.vector("dh"), T.matrix("dW")]
    r = T.rop([final], [xs, h0, W], dirs)[0]
    assert r.type == final.type


def test_structural_identity_and_document_round_trip():
    def body(x, s):
        return s * 2.0 + x
    xs, s0 = T.vector("xs"), T.scalar("s0")
    (a,), _ = scan(body, sequences=[xs], initial_states=[s0])
    (b,), _ = scan(body, sequences=[xs], initial_states=[s0])
    assert a.owner.op == b.owner.op and hash(a.owner.op) == hash(b.owner.op)
    text = T.dump_graph([xs, s0], [a])
    ins, outs, _, _ = T.load_graph(text)
    assert isinstance(outs[0].owner.op, ScanOp) and outs[0].owner.op == a.owner.op
    assert T.dump_graph(ins, outs) == text


def test_subtensor_join_shapes():
    x = T.matrix("x")
    v = T.subtensor(x, (slice(1, None, 2), 3))
    assert v.type.ndim == 1
    assert v.owner.op.infer_shape(v.owner, [(7, 5)]) == [(3,)]
    f0 = T.flip0(x)
    assert f0.owner.op.view_layout(f0.owner, [((4, 5), (5, 1), 0)]) == ((4, 5), (-5, 1), 15)
    j = T.join(0, x, x)
    assert j.owner.op.infer_shape(j.owner, [(2, 5), (3, 5)]) == [(5, 5)]
    with pytest.raises(TypeMismatch):
        T.join(0, x, T.vector("v"))


def test_loop_rewrites_last_step_and_pushout():
    from paper_1605_02688_b200.graph import FunctionGraph
    from paper_1605_02688_b200.rewrite import run_preset
    from paper_1605_02688_b200.scan import LAST
    xs = T.vector("xs")
    (hist,), _ = scan(lambda x, s: s + x, sequences=[xs], initial_states=[T.as_variable(0.0)])
    fg = FunctionGraph([xs], [hist[-1] * 2.0])
    _, log = run_preset(fg, "fast_run")
    assert log.count(rewrite="loop_last_step_only") == 1
    assert next(n for n in fg.toposort() if isinstance(n.op, ScanOp)).op.retention == (LAST,)
    for out in (T.sum(hist), hist[-1] + T.sum(hist)):   # whole history consumed: keep it
        fg = FunctionGraph([xs], [out])
        run_preset(fg, "fast_run")
        assert next(n for n in fg.toposort() if isinstance(n.op, ScanOp)).op.retention == ("full",)
    w = T.scalar("w")
    (h2,), _ = scan(lambda x, s, w_: s + x * T.exp(w_), sequences=[xs], initial_states=[T.as_variable(0.0)],
                    non_sequences=[w])
    fg = FunctionGraph([xs, w], [h2])
    _, log = run_preset(fg, "fast_run")
    assert log.count(rewrite="loop_pushout_invariants") == 1
    loop = next(n for n in fg.toposort() if isinstance(n.op, ScanOp))
    assert not any(getattr(n.op, "kernel", None) == "exp" for n in loop.op._order)
    (h3,), _ = scan(lambda x, s: s * x, sequences=[xs], initial_states=[T.as_variable(1.0)])
    fg = FunctionGraph([xs], [h3])
    _, log = run_preset(fg, "fast_run")
    assert log.count(rewrite="loop_pushout_invariants") == 0


def test_loop_rewrites_move_work_out_of_lstm_loops():
    """Graph-level check of the loop rewrites on the PTB LSTM training step
    (no device): the forward loop keeps only h.Wh and the gate composite's
    inputs, the BPTT loop only the adjoint recurrence; the input projections,
    logits, softmax / cross-entropy and the weight-gradient accumulations run
    outside as seq_dot / seq_gram products."""
    from paper_1605_02688_b200.graph import FunctionGraph, Variable, ancestor_vars, clone_outputs
    from paper_1605_02688_b200.rewrite import RewriteContext, run_preset
    from paper_1605_02688_b200.scan import SeqDot, SeqGram
    from paper_1605_02688_b200.shared import SharedVariable
    from tools.lstm_bench import build
    captured = {}
    real = T.compile

    def capture(inputs, outputs, updates=(), **kw):
        captured["args"] = (inputs, outputs, updates)
    T.compile = capture
    try:
        build(T, 16, 5, B=3, V=20)
    finally:
        T.compile = real
    inputs, outputs, updates = captured["args"]
    outs = list(outputs) + [u for _, u in updates]
    shared = sorted({v for v in ancestor_vars(outs) if isinstance(v, SharedVariable)}, key=lambda v: v.id)
    repl = {v: Variable(v.type, v.name) for v in list(inputs) + shared}
    cloned, _ = clone_outputs(outs, repl)
    fg = FunctionGraph([repl[v] for v in list(inputs) + shared], cloned)
    run_preset(fg, "fast_run", ctx=RewriteContext(execution_bound=True))
    nodes = fg.toposort()
    loops = [n.op for n in nodes if isinstance(n.op, ScanOp)]
    assert len(loops) == 2 and all(op.n_states == 2 for op in loops)
    fwd = min(loops, key=lambda op: len(op._order))
    assert sum(n.op.name == "dot" for n in fwd._order) == 1          # h . Wh only
    assert sum(isinstance(n.op, SeqDot) for n in nodes) >= 3
    assert sum(isinstance(n.op, SeqGram) for n in nodes) >= 2
