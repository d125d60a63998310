"""The CPU oracle is pinned to the real reference: every golden vector in
tests/golden/texpr_goldens.npz (produced by running texpr itself, see
make_golden.py) is reproduced bit-exactly by oracle/texpr_numpy.py, which
issues the same NumPy calls in the same order."""
import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C
from oracle import texpr_numpy as O

BINARY = ("add", "sub", "mul", "div", "pow", "maximum", "lt", "gt", "le", "ge", "eq", "neq", "second")
UNARY = ("neg", "exp", "log", "log1p", "sqr", "sqrt", "sigmoid", "tanh", "isnan")


def same(a, b):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b))
    assert np.asarray(a).dtype == np.asarray(b).dtype or np.asarray(a).dtype.kind == np.asarray(b).dtype.kind


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_elementwise_kernels_bit_exact(golden, dt):
    a, b, c = golden[f"ew_{dt}_a"], golden[f"ew_{dt}_b"], golden[f"ew_{dt}_c"]
    for k in BINARY:
        same(O.elemwise(k, [a, b]), golden[f"ew_{dt}_{k}"])
    for k in UNARY:
        same(O.elemwise(k, [a]), golden[f"ew_{dt}_{k}"])
    same(O.elemwise("switch", [c, a, b]), golden[f"ew_{dt}_switch"])


def test_integer_kernels(golden):
    a, b = golden["ew_int64_a"], golden["ew_int64_b"]
    for k in ("add", "sub", "mul", "div", "maximum", "lt", "eq"):
        same(O.elemwise(k, [a, b]), golden[f"ew_int64_{k}"])
    with pytest.raises(ZeroDivisionError):
        O.elemwise("div", [a, np.zeros_like(b)])


def test_reductions_bit_exact(golden):
    X = golden["red_X"]
    for ax in ((0,), (1,), (0, 1)):
        tag = "".join(map(str, ax))
        same(O.reduce_sum(X, ax), golden[f"red_sum_{tag}"])
        same(O.reduce_max(X, ax), golden[f"red_max_{tag}"])
        same(O.argmax_onehot(X, ax), golden[f"red_argmax_onehot_{tag}"])
    X3 = golden["red3_X"]
    for ax in ((0, 2), (1,), (0, 1, 2), (2,), (0,)):
        tag = "".join(map(str, ax))
        same(O.reduce_sum(X3, ax), golden[f"red3_sum_{tag}"])
        same(O.reduce_max(X3, ax), golden[f"red3_max_{tag}"])
        same(O.argmax_onehot(X3, ax), golden[f"red3_argmax_onehot_{tag}"])


def test_argmax_index_matches_onehot(golden):
    X = golden["red_X"]
    for ax in ((0,), (1,)):
        idx = O.argmax_index(X, ax)
        oh = O.argmax_onehot(X, ax)
        assert np.array_equal(np.argmax(np.moveaxis(oh, ax[0], -1), axis=-1), idx)


def test_dot(golden):
    A, B, v = golden["dot_A"], golden["dot_B"], golden["dot_v"]
    same(O.dot(A, B), golden["dot_mm"])
    same(O.dot(A, v), golden["dot_mv"])
    same(O.dot(v, B), golden["dot_vm"])
    same(O.dot(v, v), golden["dot_vv"])
    same(O.dot(A.T, A), golden["dot_tn"])


def _cfg2_inputs():
    r7 = np.random.default_rng(7)
    return [r7.standard_normal(40000, dtype=np.float32) for _ in range(4)]


def test_config2_interpreter_fused_and_unfused(golden):
    ins = _cfg2_inputs()
    g = C.build_ew(T)
    fused = C.CpuFunction(T, g["inputs"], g["outputs"], preset="fast_run")
    assert len(fused.fg.toposort()) == 1  # one composite, as in the reference
    same(fused(*ins), golden["cfg2_fused"])
    plain = C.CpuFunction(T, g["inputs"], g["outputs"], preset="none")
    same(plain(*ins), golden["cfg2_unfused"])


def test_config1_logreg_steps(golden):
    x, y = C.inputs_logreg()
    g = C.build_logreg(T)
    f = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"], preset="fast_run", exclude=("fuse_elemwise",))
    assert len(f.fg.toposort()) == int(golden["cfg1_nodes"]) == 45
    costs = [f(x, y)[0] for _ in range(3)]
    same(np.array(costs), golden["cfg1_costs"])
    W, b = g["params"]
    same(f.value(W), golden["cfg1_W"])
    same(f.value(b), golden["cfg1_b"])
    assert abs(costs[0] - np.log(10)) < 1e-6


def test_config4_small_mlp_steps(golden):
    B, H = 64, 96
    g = C.build_mlp(T, B=B, H=H)
    x, y = C.inputs_mlp(B=B)
    f = C.CpuFunction(T, g["inputs"], g["outputs"], g["updates"], preset="fast_run", exclude=("fuse_elemwise",))
    assert len(f.fg.toposort()) == int(golden["cfg4_nodes"])
    costs = np.array([f(x, y)[0] for _ in range(2)])
    same(costs, golden["cfg4_costs"])
    for i, p in enumerate(g["params"]):
        same(f.value(p), golden[f"cfg4_p{i}"])
