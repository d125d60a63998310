"""Runtime semantics of the device VM, mirroring the reference's
tests/test_runtime.py (compile/call, shared state, updates, broadcast
enforcement, copies) plus CUDA-graph replay and device-tensor calls."""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from paper_1605_02688_b200.errors import ShapeMismatch, TypeMismatch, UnderdeterminedOutputs

pytestmark = pytest.mark.gpu


def test_compile_and_call_basic():
    x = T.vector("x")
    f = T.compile([x], [x + 1.0], preset="none")
    np.testing.assert_array_equal(f([1.0, 2.0])[0], [2.0, 3.0])


def test_single_output_convenience():
    x = T.scalar("x")
    f = T.compile([x], x * 2.0, preset="none")
    assert float(f(3.0)) == 6.0


def test_compile_from_intermediate_skips_producers(rng):
    x = T.vector("x")
    h = T.exp(x)
    y = T.sum(h * 2.0)
    f = T.compile([h], y, preset="none")
    assert all(getattr(n.op, "kernel", "") != "exp" for n in f.order)
    hv = rng.standard_normal(4)
    assert float(f(hv)) == pytest.approx(float(np.sum(hv * 2.0)))


def test_underdetermined_outputs_rejected():
    x, y = T.vector("x"), T.vector("y")
    with pytest.raises(UnderdeterminedOutputs):
        T.compile([x], [x + y], preset="none")


def test_shared_updates_counter():
    s = T.shared(np.array(0.0), name="s")
    f = T.compile([], [s], updates=[(s, s + 1.0)], preset="none")
    outs = [float(f()[0]) for _ in range(3)]
    assert outs == [0.0, 1.0, 2.0]  # outputs see the value before the update
    assert float(s.get_value()) == 3.0


def test_update_in_place_when_safe():
    W = T.shared(np.ones((64, 32), np.float32), name="W")
    x = T.matrix("x", dtype="float32")
    y = T.sum(T.dot(x, W))
    f = T.compile([x], [y], updates=[(W, W - 0.5 * W)])
    xv = np.ones((4, 64), np.float32)
    assert float(f(xv)[0]) == 4 * 32 * 64
    assert float(f(xv)[0]) == 4 * 32 * 64 * 0.5
    np.testing.assert_array_equal(W.get_value(), np.full((64, 32), 0.25, np.float32))


def test_swap_updates_read_old_values():
    a = T.shared(np.array([1.0, 2.0]), name="a")
    b = T.shared(np.array([3.0, 4.0]), name="b")
    f = T.compile([], [], updates=[(a, b), (b, a)])
    f()
    np.testing.assert_array_equal(a.get_value(), [3.0, 4.0])
    np.testing.assert_array_equal(b.get_value(), [1.0, 2.0])


def test_updates_may_reference_outputs():
    s = T.shared(np.zeros(3), name="s")
    x = T.vector("x")
    y = x * 2.0
    f = T.compile([x], [y], updates=[(s, s + y)])
    f([1.0, 2.0, 3.0])
    out = f([1.0, 1.0, 1.0])
    np.testing.assert_array_equal(out[0], [2.0, 2.0, 2.0])
    np.testing.assert_array_equal(s.get_value(), [4.0, 6.0, 8.0])


def test_two_functions_same_region_coexist(rng):
    x = T.vector("x")
    h = T.tanh(x)
    f1 = T.compile([x], T.sum(h))
    f2 = T.compile([x], T.sum(h * h))
    p = rng.standard_normal(5)
    assert float(f1(p)) == pytest.approx(float(np.sum(np.tanh(p))))
    assert float(f2(p)) == pytest.approx(float(np.sum(np.tanh(p) ** 2)))


def test_update_pair_type_checked():
    s = T.shared(np.zeros(3), name="s")
    bad = T.scalar("b")
    with pytest.raises(TypeMismatch):
        T.compile([bad], [bad], updates=[(s, bad)])


def test_broadcastable_dims_enforced_at_call():
    x = T.make_input(T.TensorType("float64", (True, False)), "x")
    f = T.compile([x], [x * 2.0])
    f(np.zeros((1, 4)))
    with pytest.raises(TypeMismatch):
        f(np.zeros((3, 4)))


def test_runtime_broadcast_requires_declaration():
    x, y = T.matrix("x"), T.matrix("y")
    f = T.compile([x, y], x + y)
    with pytest.raises(ShapeMismatch):
        f(np.zeros((3, 4)), np.zeros((1, 4)))


def test_wrong_dtype_rejected():
    x = T.vector("x", dtype="float64")
    f = T.compile([x], [x + 1.0])
    with pytest.raises(TypeMismatch):
        f(np.array(["a", "b"], dtype=object))


def test_shared_set_value_and_shape_change():
    s = T.shared(np.zeros(3, np.float32), name="s")
    f = T.compile([], [s * 2.0])
    np.testing.assert_array_equal(f()[0], [0, 0, 0])
    s.set_value(np.ones(3, np.float32))
    np.testing.assert_array_equal(f()[0], [2, 2, 2])
    s.set_value(np.arange(5, dtype=np.float32))
    np.testing.assert_array_equal(f()[0], 2 * np.arange(5, dtype=np.float32))
    with pytest.raises(TypeMismatch):
        s.set_value(np.zeros((2, 2)))


def test_graph_replay_is_stable(rng):
    x = T.matrix("x", dtype="float32")
    f = T.compile([x], [T.sum(T.exp(x) * 2.0, axis=1), T.max(x)])
    xv = rng.standard_normal((100, 37)).astype(np.float32)
    first = f(xv)
    for _ in range(5):
        again = f(xv)
        for a, b in zip(first, again):
            np.testing.assert_array_equal(a, b)
    assert f.profile.call_count == 6


def test_call_device_with_torch_tensors(rng):
    import torch
    x = T.vector("x", dtype="float32")
    f = T.compile([x], [T.sqr(x) + 1.0])
    xv = torch.from_numpy(rng.standard_normal(1000).astype(np.float32)).cuda()
    (y,) = f.call_device(xv, sync=True)
    assert y.is_cuda
    np.testing.assert_allclose(y.cpu().numpy(), xv.cpu().numpy() ** 2 + 1.0, rtol=1e-6)


def test_copy_with_swap():
    s = T.shared(np.array(1.0), name="s")
    s2 = T.shared(np.array(10.0), name="s2")
    f = T.compile([], [s], updates=[(s, s * 2.0)])
    g = f.copy(swap={s: s2})
    g()
    assert float(s2.get_value()) == 20.0 and float(s.get_value()) == 1.0
    h = f.copy(carry_updates=False)
    h()
    assert float(s.get_value()) == 1.0


def test_profile_nodes_records_times(rng):
    x = T.matrix("x", dtype="float32")
    f = T.compile([x], [T.sum(T.tanh(x), axis=0)])
    f.profile_nodes = True
    f(rng.standard_normal((64, 64)).astype(np.float32))
    assert all(f.profile.node_calls[n.id] == 1 for n in f.order)
    assert sum(f.profile.node_time.values()) > 0


# -- chunk-pipelined host calls (stream.py) ------------------------------------

def _pipe_used(f):
    return any(p for p in f._pipes.values())


def test_pipelined_host_call_matches_device_call_ragged():
    """Host inputs above stream.MIN_BYTES run as overlapped H2D/compute/D2H
    chunks; results must be bit-identical to the single-plan device call,
    including a ragged last chunk."""
    import torch
    from oracle import configs as C
    from oracle import texpr_numpy as O
    g = C.build_ew(T)
    f = T.compile(g["inputs"], g["outputs"])
    n = (1 << 24) + 77
    ins = C.inputs_ew(n, seed=7)
    got = f(*ins)
    assert _pipe_used(f)
    dev = f.call_device(*[torch.from_numpy(a).cuda() for a in ins], sync=True).cpu().numpy()
    np.testing.assert_array_equal(got, dev)
    idx = np.random.default_rng(0).integers(0, n, 4096)
    want = O.eval_composite_plain(f.order[0].op.program, [a[idx] for a in ins])[0]
    np.testing.assert_allclose(got[idx], want, rtol=1e-5, atol=1e-6)
    # pinned torch inputs take the same path; a second call reuses the slots
    pins = [torch.from_numpy(a).pin_memory() for a in ins]
    np.testing.assert_array_equal(f(*pins), dev)


def test_pipelined_multi_output_matrix_and_bool():
    a, b = T.matrix("a", dtype="float32"), T.matrix("b", dtype="float32")
    f = T.compile([a, b], [T.tanh(a) * b, T.gt(a, b), a - b])
    rng = np.random.default_rng(3)
    av = rng.standard_normal((4099, 4096), dtype=np.float32)
    bv = rng.standard_normal((4099, 4096), dtype=np.float32)
    o1, o2, o3 = f(av, bv)
    assert _pipe_used(f)
    assert o2.dtype == np.bool_ and o2.shape == av.shape
    np.testing.assert_array_equal(o2, av > bv)
    np.testing.assert_array_equal(o3, av - bv)
    np.testing.assert_allclose(o1, np.tanh(av) * bv, rtol=1e-5, atol=1e-6)


def test_pipelined_integer_division_by_zero_raises():
    a, b = T.vector("a", dtype="int32"), T.vector("b", dtype="int32")
    f = T.compile([a, b], a / b)  # integer div floors and raises on zero (ops/elemwise.py:49-55)
    av = np.ones(1 << 25, np.int32)
    bv = np.ones(1 << 25, np.int32)
    bv[-5] = 0
    with pytest.raises(ZeroDivisionError):
        f(av, bv)


# -- NaN guard (reference diagnostics.py:52-88; test_runtime.py:137-153) -------------

def test_nan_guard_failed_call_leaves_shared_untouched():
    s = T.shared(np.array(10.0), name="s")
    x = T.vector("x")
    f = T.compile([x], [T.sum(T.log(x))], updates=[(s, s + 1.0)], preset="none", nan_guard=T.NanGuardConfig())
    f(np.array([1.0, 2.0]))
    assert float(s.get_value()) == 11.0
    from paper_1605_02688_b200.errors import NanDetected
    with pytest.raises(NanDetected) as e:
        f(np.array([-1.0, 2.0]))
    assert float(s.get_value()) == 11.0   # unchanged by the failed call
    r = e.value.report
    assert r.check == "nan" and r.op == "log" and r.tensor == "output 0" and "shape (2,)" in r.value_summary
    f(np.array([3.0, 2.0]))
    assert float(s.get_value()) == 12.0


def test_nan_guard_inf_big_and_inputs():
    from paper_1605_02688_b200.errors import NanDetected
    x = T.vector("x", dtype="float32")
    f = T.compile([x], [T.exp(x) * 2.0], nan_guard=T.NanGuardConfig(big_threshold=1e6))
    np.testing.assert_allclose(f(np.array([0.0, 1.0], np.float32))[0], [2.0, 2 * np.e], rtol=1e-6)
    with pytest.raises(NanDetected) as e:
        f(np.array([20.0, 0.0], np.float32))        # exp(20) = 4.9e8 > 1e6
    assert e.value.report.check == "big"
    with pytest.raises(NanDetected) as e:
        f(np.array([100.0, 0.0], np.float32))       # exp overflows to inf
    assert e.value.report.check == "inf"
    with pytest.raises(NanDetected) as e:
        f(np.array([np.nan, 0.0], np.float32))      # caught at the first node, on its input
    assert e.value.report.check == "nan" and e.value.report.tensor == "input 0"
    g = T.compile([x], [T.exp(x)], nan_guard=T.NanGuardConfig(check_inf=False, big_threshold=None))
    assert np.isinf(g(np.array([100.0], np.float32))[0][0])


# -- lazy conditional and breakpoint (reference test_runtime.py:84-131, test_ops.py:295-349) --

def _lazy_fixture():
    c, p = T.scalar("c"), T.vector("p")
    expensive = T.exp(T.sqr(p)) * 3.0
    cheap = p + 1.0
    out = T.ifelse(c > 0.0, T.sum(expensive), T.sum(cheap))
    f = T.compile([c, p], [out], preset="none")
    roots = {True: next(n for n in f.order if getattr(n.op, "kernel", "") == "exp"),
             False: next(n for n in f.order if getattr(n.op, "kernel", "") == "add")}
    return f, roots


def test_ifelse_untaken_branch_never_runs(rng):
    f, roots = _lazy_fixture()
    point = rng.standard_normal(4)
    np.testing.assert_allclose(f(-1.0, point)[0], np.sum(point + 1.0), rtol=1e-12)
    assert f.profile.node_calls.get(roots[True].id, 0) == 0
    assert f.profile.node_calls.get(roots[False].id, 0) == 1
    np.testing.assert_allclose(f(1.0, point)[0], np.sum(np.exp(point ** 2) * 3.0), rtol=1e-12)
    assert f.profile.node_calls.get(roots[True].id, 0) == 1


def test_ifelse_randomized_conditions_and_values(rng):
    f, roots = _lazy_fixture()
    taken = 0
    for _ in range(30):
        c = float(rng.standard_normal())
        before = f.profile.node_calls.get(roots[True].id, 0)
        f(c, rng.standard_normal(4))
        assert f.profile.node_calls.get(roots[True].id, 0) - before == (1 if c > 0 else 0)
        taken += c > 0
    assert 0 < taken < 30
    c, a, b = T.scalar("c"), T.vector("a"), T.vector("b")
    g = T.compile([c, a, b], [T.ifelse(c > 0.0, a * 2.0, b * 3.0)], preset="none")
    av, bv = rng.standard_normal(3), rng.standard_normal(3)
    np.testing.assert_array_equal(g(1.0, av, bv)[0], av * 2.0)
    np.testing.assert_array_equal(g(-1.0, av, bv)[0], bv * 3.0)


def test_ifelse_gradient_and_updates(rng):
    c, x = T.scalar("c"), T.vector("x")
    w = T.shared(np.array([1.0, 2.0, 3.0]), name="w")
    y = T.ifelse(c > 0.0, T.sum(w * x), T.sum(w * w))
    gw = T.grad(y, w)
    f = T.compile([c, x], [y, gw], updates=[(w, w - 0.1 * gw)])
    xv = np.array([0.5, -1.0, 2.0])
    yv, gv = f(1.0, xv)
    assert float(yv) == pytest.approx(float(np.dot([1.0, 2.0, 3.0], xv)))
    np.testing.assert_allclose(gv, xv)
    np.testing.assert_allclose(w.get_value(), np.array([1.0, 2.0, 3.0]) - 0.1 * xv)


def test_breakpoint_fires_passes_through_and_aborts():
    from paper_1605_02688_b200.errors import BreakpointAbort
    calls = []
    T.register_breakpoint_handler("d1", lambda names, values: calls.append((names, [v.copy() for v in values])))
    x = T.vector("x")
    (mon,) = T.breakpoint_op(T.max(T.isnan(x)), [x], label="d1")
    f = T.compile([x], [mon], preset="none")
    np.testing.assert_array_equal(f(np.array([1.0, 2.0]))[0], [1.0, 2.0])
    assert calls == []
    v = np.array([1.0, np.nan, 3.0])
    np.testing.assert_array_equal(f(v)[0], v)
    assert len(calls) == 1 and np.array_equal(calls[0][1][0], v, equal_nan=True)
    T.register_breakpoint_handler("d1", None)
    s = T.shared(np.array(0.0), name="s")
    T.register_breakpoint_handler("d3", lambda names, values: "abort")
    y = T.scalar("y")
    (m2,) = T.breakpoint_op(y > 0.0, [y], label="d3")
    g = T.compile([y], [m2], updates=[(s, s + 1.0)], preset="none")
    assert float(g(-1.0)[0]) == -1.0 and float(s.get_value()) == 1.0
    with pytest.raises(BreakpointAbort):
        g(1.0)
    assert float(s.get_value()) == 1.0      # aborted call committed nothing
    T.register_breakpoint_handler("d3", None)


def test_allow_gc_is_bit_exact(rng):
    """reference test_runtime.py:177-186: keeping intermediates changes memory
    use, never values (the device arena is planned once either way)."""
    x = T.matrix("x", dtype="float32")
    e = T.tanh(T.dot(x, x.T) * 0.5) - T.dimshuffle(T.sum(x, axis=1), (0, "x"))
    v = rng.standard_normal((64, 48)).astype(np.float32)
    a = T.compile([x], e, allow_gc=True)(v)
    b = T.compile([x], e, allow_gc=False)(v)
    assert np.array_equal(a, b)


def test_no_device_allocations_after_the_second_call(rng):
    """reference test_runtime.py:189-203 (zero node-output allocations on the
    2nd call): after planning and graph capture a training step allocates
    nothing on the device."""
    import torch
    from oracle import configs as C
    g = C.build_mlp(T, B=256, H=128)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    x, y = C.inputs_mlp(B=256)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for _ in range(3):
        f.call_device(xd, yd, sync=True)
    before = torch.cuda.memory_allocated()
    for _ in range(5):
        f.call_device(xd, yd, sync=True)
    assert torch.cuda.memory_allocated() == before


def test_device_fault_leaves_updates_uncommitted():
    """reference test_runtime.py:137-171 (a failing node leaves shared state
    untouched): an integer division by zero detected on the device fails the
    call before the update is written back."""
    s = T.shared(np.arange(6, dtype=np.int64), name="s")
    a = T.vector("a", dtype="int64")
    b = T.vector("b", dtype="int64")
    from paper_1605_02688_b200.elemwise import make
    q = make("div", [a, b])  # integer div floors, and flags a zero divisor on the device
    f = T.compile([a, b], [q], updates=[(s, s + q)])
    f(np.full(6, 7, np.int64), np.full(6, 2, np.int64))
    assert np.array_equal(s.get_value(), np.arange(6) + 3)
    with pytest.raises(ZeroDivisionError):
        f(np.full(6, 7, np.int64), np.array([1, 2, 0, 4, 5, 6], np.int64))
    assert np.array_equal(s.get_value(), np.arange(6) + 3)
    f(np.full(6, 7, np.int64), np.full(6, 7, np.int64))
    assert np.array_equal(s.get_value(), np.arange(6) + 4)


def test_elementwise_never_in_place_over_a_view_of_itself(rng):
    """x * x.T where x dies at the product: writing the product into x's
    buffer would race with the transposed reads (regression found by the
    random view graphs; the result was run-to-run different)."""
    a = T.matrix("a", dtype="float32")
    b = T.matrix("b", dtype="float32")
    d = T.dot(a, b)
    f = T.compile([a, b], d * T.dimshuffle(d, (1, 0)), gemm_mode="simt")
    av = rng.standard_normal((96, 96)).astype(np.float32)
    bv = rng.standard_normal((96, 96)).astype(np.float32)
    dv = av.astype(np.float64) @ bv
    want = dv * dv.T
    for _ in range(5):
        np.testing.assert_allclose(f(av, bv), want, rtol=1e-4, atol=1e-3)


def test_zero_division_flag_not_clobbered_by_reused_buffers():
    """The device zero-division flag lives for the whole step; it used to be
    placed after the liveness walk, in memory an intermediate later reused
    (a // (c*c + 1) raised ZeroDivisionError; found by the random integer
    graphs)."""
    from paper_1605_02688_b200.elemwise import make
    a, c = T.vector("a", dtype="int32"), T.vector("c", dtype="int32")
    d = make("add", [make("mul", [c, c]), T.as_variable(np.asarray(1, dtype="int64"))])
    av = np.arange(-5, 5, dtype=np.int32)
    for preset in ("none", "fast_run"):
        got = T.compile([a, c], make("div", [a, d]), preset=preset)(av, av)
        np.testing.assert_array_equal(got, av.astype(np.int64) // (av.astype(np.int64) ** 2 + 1))


def test_update_to_a_view_of_itself_and_unread_targets():
    """A <- A.T (the update value is another view of the target's own
    buffer: it used to be mistaken for an identity update and skipped),
    B <- A (B read by nothing: it used to crash the scheduler), with the
    reference's write-back-after-the-step semantics."""
    a0 = np.arange(12.0).reshape(3, 4)[:, :3].copy()
    A = T.shared(a0.copy(), name="A")
    B = T.shared(np.zeros((3, 3)), name="B")
    x = T.scalar("x")
    f = T.compile([x], T.sum(A) * x, updates=[(A, T.dimshuffle(A, (1, 0))), (B, A)])
    assert float(f(2.0)) == 2 * a0.sum()
    np.testing.assert_array_equal(A.get_value(), a0.T)
    np.testing.assert_array_equal(B.get_value(), a0)
    f(1.0)
    np.testing.assert_array_equal(A.get_value(), a0)
    np.testing.assert_array_equal(B.get_value(), a0.T)


# -- step-plan cache (shape-keyed, bounded, pointer independent) ----------------

def test_fresh_device_batches_reuse_one_plan_and_flat_memory():
    """A data loader hands a new CUDA tensor every step: the MLP step keeps one
    plan (device inputs copied into its slots), device memory stays flat and
    every step equals the same step fed by host arrays."""
    import torch
    from oracle import configs as C
    B, H = 128, 256
    ga = C.build_mlp(T, B=B, H=H)
    fa = T.compile(ga["inputs"], ga["outputs"], updates=ga["updates"])
    gb = C.build_mlp(T, B=B, H=H)
    fb = T.compile(gb["inputs"], gb["outputs"], updates=gb["updates"])
    x, y = C.inputs_mlp(B=B, seed=3)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    mem = None
    ring = []   # the loader keeps a few batches alive: addresses keep changing
    for i in range(200):
        xi, yi = torch.empty_like(xd), torch.empty_like(yd)
        xi.copy_(xd)
        yi.copy_(yd)
        ring = (ring + [(xi, yi)])[-3:]
        ca = float(fa.call_device(xi, yi, sync=True)[0].item())
        if i % 40 == 0:
            cb = float(fb(x, y)[0])
            for _ in range(39 if i < 160 else 0):
                fb(x, y)
            assert ca == cb, (i, ca, cb)
        del xi, yi
        if i == 5:
            torch.cuda.synchronize()
            mem = torch.cuda.memory_allocated()
    torch.cuda.synchronize()
    assert len(fa._plans) == 1
    assert next(iter(fa._plans.values())).slot_inputs
    assert torch.cuda.memory_allocated() <= mem


def test_plan_cache_is_bounded_lru():
    from paper_1605_02688_b200 import vm
    x = T.matrix("x", dtype="float32")
    f = T.compile([x], [T.sum(T.exp(x), axis=1)])
    outs = {}
    for r in range(1, vm.MAX_PLANS + 5):
        a = np.full((r, 3), 0.5, np.float32)
        outs[r] = f(a)[0]
        assert len(f._plans) <= vm.MAX_PLANS
    for r, o in outs.items():
        np.testing.assert_allclose(o, np.full(r, 3 * np.exp(np.float32(0.5)), np.float32), rtol=1e-6)


def test_device_outputs_survive_plan_eviction():
    """call_device returns views into the plan's arena; evicting the plan (a
    shape-changing update, LRU) must not free memory the caller still holds."""
    import torch
    s = T.shared(np.zeros(4, np.float32), name="s")
    x = T.vector("x", dtype="float32")
    f = T.compile([x], [x * 2.0 + T.sum(s)], updates=[(s, T.join(0, s, s))])
    a = torch.arange(6, dtype=torch.float32, device="cuda")
    out = f.call_device(a, sync=True)
    keep = out[0] if isinstance(out, (list, tuple)) else out
    for r in range(2, 14):
        f.call_device(torch.ones(r, device="cuda"), sync=True)
        torch.empty(1 << 20, device="cuda").fill_(7.0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(keep.cpu().numpy(), np.arange(6, dtype=np.float32) * 2.0)
    assert len(f._plans) <= 1   # plans baked on the replaced storages were dropped


def test_pipelined_identity_output_not_overwritten():
    """compile([x, y], [x, x*y]) through the chunk pipeline: the first output is
    copied out of the slot's input buffer, which the next H2D must not
    overwrite early (stream.py slot reuse)."""
    from paper_1605_02688_b200 import stream as S
    x, y = T.vector("x", dtype="float32"), T.vector("y", dtype="float32")
    f = T.compile([x, y], [x, x * y, x + y])
    n = (S.MIN_BYTES // 4) + 12345
    rng = np.random.default_rng(9)
    a = rng.standard_normal(n).astype(np.float32)
    b = rng.standard_normal(n).astype(np.float32)
    for _ in range(3):
        o0, o1, o2 = f(a, b)
        assert _pipe_used(f)
        np.testing.assert_array_equal(o0, a)
        np.testing.assert_array_equal(o1, a * b)
        np.testing.assert_array_equal(o2, a + b)


def test_user_plugin_op_with_host_perform_runs_as_host_step():
    """An op written against the reference's plugin contract only (host
    ``perform``, no device lowering, no infer_shape) still executes: as a host
    step between device launches, shapes probed from one host evaluation."""
    from paper_1605_02688_b200.graph import apply
    from paper_1605_02688_b200.op import Op, is_host_op

    class HostCube(Op):
        name = "host_cube_fixture"

        def infer_types(self, input_types):
            return [input_types[0]]

        def perform(self, inputs, output_buffers=None):
            return [inputs[0] ** 3]

        def grad(self, inputs, output_grads):
            return [output_grads[0] * 3.0 * inputs[0] * inputs[0]]

    assert is_host_op(HostCube())
    x = T.vector("x", dtype="float64")
    y = T.exp(apply(HostCube(), [T.tanh(x)])[0]) * 2.0
    (g,) = T.grad(T.sum(y), [x])
    f = T.compile([x], [y, g])
    xv = np.linspace(-1, 1, 7)
    yv, gv = f(xv)
    t = np.tanh(xv)
    np.testing.assert_allclose(yv, np.exp(t ** 3) * 2.0, rtol=1e-12)
    np.testing.assert_allclose(gv, np.exp(t ** 3) * 2.0 * 3 * t * t * (1 - t * t), rtol=1e-12)
    plan = next(iter(f._plans.values()))
    assert plan.host_ops == 1 and plan.graph is None
    rep = T.verify_grad([x], [y], [xv], rel_tol=1e-6)
    assert rep.passed, str(rep)


def test_host_plugin_op_inside_a_loop_body():
    """A perform-only plugin op inside a scan body: the loop's step plans and
    the enclosing step run eagerly (no graph capture), results match."""
    from paper_1605_02688_b200.graph import apply
    from paper_1605_02688_b200.op import Op

    class HostHalf(Op):
        name = "host_half_fixture"

        def infer_types(self, input_types):
            return [input_types[0]]

        def perform(self, inputs, output_buffers=None):
            return [inputs[0] * 0.5]

    xs = T.matrix("xs", dtype="float64")
    h0 = T.vector("h0", dtype="float64")
    hist, _ = T.scan(lambda x, h: apply(HostHalf(), [T.tanh(h + x)])[0], sequences=[xs], initial_states=[h0])
    out = hist[0] if isinstance(hist, (list, tuple)) else hist
    f = T.compile([xs, h0], [out])
    xv = np.random.default_rng(1).standard_normal((5, 3))
    got = f(xv, np.zeros(3))[0]
    h, want = np.zeros(3), []
    for t in range(5):
        h = np.tanh(h + xv[t]) * 0.5
        want.append(h)
    np.testing.assert_allclose(got, np.array(want), rtol=1e-12)
    for _ in range(2):
        np.testing.assert_allclose(f(xv, np.zeros(3))[0], np.array(want), rtol=1e-12)
    assert next(iter(f._plans.values())).graph is None


@pytest.mark.parametrize("regions", [
    (((None, None, None), (0, 3, None)), ((None, None, None), (3, 5, None)), ((None, None, None), (5, 8, None))),
    (((None, None, None), (0, 3, None)), ((None, None, None), (5, 8, None))),            # a gap: zero-filled
    (((None, None, None), (0, 5, None)), ((None, None, None), (3, 8, None))),            # overlap: summed
])
def test_zero_embed_placement_and_fallback(regions):
    """ZeroEmbed (the LSTM's gate-gradient assembly): a partition has its
    producers write straight into their regions; gaps and overlaps take the
    zero-fill + add path.  Values equal the inc_subtensor chain over zeros."""
    from paper_1605_02688_b200.graph import apply
    from paper_1605_02688_b200.shaping import ZeroEmbed
    x = T.matrix("x", dtype="float64")
    vals = [T.matrix(f"v{k}", dtype="float64") for k in range(len(regions))]
    ze = apply(ZeroEmbed(regions), [x] + [T.tanh(v) * 2.0 for v in vals])[0]
    f = T.compile([x] + vals, [ze * 1.0 + 0.0])
    rng = np.random.default_rng(3)
    xv = rng.standard_normal((4, 8))
    vv = [rng.standard_normal((4, r[1][1] - r[1][0])) for r in regions]
    got = f(xv, *vv)[0]
    want = np.zeros((4, 8))
    for r, v in zip(regions, vv):
        want[:, r[1][0]:r[1][1]] += np.tanh(v) * 2.0
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-15)
    plan = next(iter(f._plans.values()))
    ze_nodes = [n for n in f.order if n.op.name == "zero_embed"]
    assert ze_nodes
    assert bool(plan.placed.get(ze_nodes[0].id)) == (len(regions) == 3)
    # its portable (reference-op) form round-trips through a saved container
    g = T.load(f.save())
    np.testing.assert_allclose(g(xv, *vv)[0], want, rtol=1e-12, atol=1e-15)
