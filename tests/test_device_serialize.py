"""Function containers on the device: files written by the reference run on
the B200 and continue the reference's own trajectory; this package's
containers resume training exactly (checkpoint / resume).
Reference files and expectations come from tests/golden/make_txfn.py."""
import os

import numpy as np
import pytest

import paper_1605_02688_b200 as T
from oracle import configs as C

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _read(name):
    return open(os.path.join(GOLD, name), "rb").read()


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(np.asarray(b, np.float64)), 1e-30))


def test_reference_logreg_checkpoint_continues_on_device():
    exp = np.load(os.path.join(GOLD, "ref_txfn_expect.npz"))
    f = T.load(_read("ref_logreg_after2.txfn"))
    x, y = C.inputs_logreg(N=600)
    cost3 = float(f(x, y)[0])
    assert abs(cost3 - float(exp["logreg_costs"][2])) <= 1e-5 * abs(float(exp["logreg_costs"][2]))
    sh = {s.name: s for s, _ in f.shared_bindings}
    assert _rel(sh["W"].get_value(), exp["logreg_W3"]) <= 1e-5
    assert _rel(sh["b"].get_value(), exp["logreg_b3"]) <= 1e-5


def test_reference_ew_container_on_device():
    exp = np.load(os.path.join(GOLD, "ref_txfn_expect.npz"))
    f = T.load(_read("ref_ew.txfn"))
    got = f(*C.inputs_ew(1000, seed=5))
    np.testing.assert_allclose(got, exp["ew_out"], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("reopt", [False, True])
def test_save_load_resumes_training_bit_exact(reopt):
    """MLP (TF32 GEMMs, fused epilogues): 2 steps, save, then one more step on
    the original and on the loaded copy -- identical costs and parameters."""
    B, H = 256, 512
    x, y = C.inputs_mlp(B=B)
    g = C.build_mlp(T, B=B, H=H)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"])
    for _ in range(2):
        f(x, y)
    blob = f.save()
    h = T.load(blob, force_reoptimize=reopt)
    c_orig, c_load = f(x, y)[0], h(x, y)[0]
    assert c_orig == c_load
    orig = {s.name: s.get_value() for s, _ in f.shared_bindings}
    for s, _ in h.shared_bindings:
        assert np.array_equal(s.get_value(), orig[s.name]), s.name
    # without re-optimisation the loaded function saves to the same bytes
    if not reopt:
        assert T.save(h) == T.save(f)


def test_saved_values_are_device_state():
    W = T.shared(np.zeros((4, 3), np.float32), name="W")
    x = T.matrix("x", dtype="float32")
    f = T.compile([x], T.sum(T.dot(x, W)), updates=[(W, W + 1.0)])
    f(np.ones((2, 4), np.float32))
    f(np.ones((2, 4), np.float32))
    g = T.load(f.save())
    (s, _), = g.shared_bindings
    np.testing.assert_array_equal(s.get_value(), np.full((4, 3), 2.0, np.float32))
    assert float(g(np.ones((2, 4), np.float32))) == 2 * 3 * 4 * 2.0


@pytest.mark.parametrize("reopt", [False, True])
def test_data_parallel_step_resumes_from_checkpoint(reopt):
    """A saved MLP step loads with data_parallel (no update fused into a
    gradient GEMM, since gradients are partial sums until the allreduce) and
    continues exactly like the data-parallel step it was saved from."""
    from paper_1605_02688_b200.dp import DataParallel
    B, H = 128, 256
    x, y = C.inputs_mlp(B=B)
    g = C.build_mlp(T, B=B, H=H)
    f = T.compile(g["inputs"], g["outputs"], updates=g["updates"], data_parallel=DataParallel(world_size=1, rank=0))
    f(x, y)
    blob = f.save()
    h = T.load(blob, force_reoptimize=reopt, data_parallel=DataParallel(world_size=1, rank=0))
    assert h.shard is not None and len(h.shard.partial_vars) >= 6
    c_orig, c_load = float(f(x, y)[0]), float(h(x, y)[0])
    assert abs(c_orig - c_load) <= 1e-6 * abs(c_orig)
    orig = {s.name: s.get_value() for s, _ in f.shared_bindings}
    for s, _ in h.shared_bindings:
        assert _rel(s.get_value(), orig[s.name]) <= 1e-6, s.name
