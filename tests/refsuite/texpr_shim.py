"""pytest plugin: run the REFERENCE's own test files against this package.

``import texpr`` (and every ``texpr.*`` submodule the reference tests import)
resolves to ``paper_1605_02688_b200``: the drop-in claim checked by the
reference's own assertions (VERDICT r1 "next" #5).

Used by ``tools/run_reference_suite.sh`` as ``pytest -p texpr_shim`` over a
git-ignored copy of ``/root/reference/pkg/tests`` (``baseline/_ref_tests``;
the reference sources are never committed).  Two reference modules have no
device counterpart and are supplied here from test infrastructure:

* ``texpr.interp.eval_graph``: the reference's host interpreter -- the tests
  use it as their expected-value oracle -- is the repo's NumPy restatement
  (``oracle/texpr_numpy.evaluate``, which follows ``interp.py:20-51``);
* ``texpr.testing``: the reference's random-graph generator, loaded from the
  installed reference (``baseline/_ref/texpr/testing.py``) so that it builds
  its graphs through THIS package's front end.

``texpr.alloc.track_allocations`` inspects the reference's host allocator
(``alloc.py``); the device VM plans one arena per shape and has no per-call
host allocations to count, so tests entering it are skipped with that reason.
"""
from __future__ import annotations

import contextlib
import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import pytest  # noqa: E402

import paper_1605_02688_b200 as P  # noqa: E402


def _m(name):
    # submodules by import (package attributes may be shadowed: P.scan is the function)
    return importlib.import_module("paper_1605_02688_b200." + name)


graph = _m("graph")


def _interp():
    from oracle import texpr_numpy as O
    m = types.ModuleType("texpr.interp")

    def eval_graph(outputs, bindings=None, check_shapes=True):
        """interp.eval_graph (interp.py:20-51): the NumPy oracle per node,
        after this package's own runtime shape check of the node
        (``op.check_runtime_shapes``, the reference's ops/base.py:132-163)."""
        import numpy as np
        outputs = list(outputs)
        env = {v.id: np.asarray(a, dtype=np.dtype(v.type.dtype)) for v, a in dict(bindings or {}).items()}
        for node in graph.io_toposort(outputs):
            args = [env[x.id] if x.id in env else np.asarray(x.value) for x in node.inputs]
            if check_shapes:
                node.op.check_runtime_shapes(node, [a.shape for a in args])
            for o, r in zip(node.outputs, O.run_node(node, args)):
                env[o.id] = np.asarray(r)
        return [env[v.id] if v.id in env else np.asarray(v.value) for v in outputs]
    m.eval_graph = eval_graph
    return m


def _alloc():
    m = types.ModuleType("texpr.alloc")

    @contextlib.contextmanager
    def track_allocations():
        pytest.skip("host allocator introspection (reference alloc.py) has no device counterpart: "
                    "the VM plans one liveness arena per shape signature")
        yield None
    m.track_allocations = track_allocations
    return m


def _testing():
    path = os.path.join(ROOT, "baseline", "_ref", "texpr", "testing.py")
    spec = importlib.util.spec_from_file_location("texpr.testing", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules["texpr.testing"] = mod
    spec.loader.exec_module(mod)
    return mod


def install():
    mods = {
        "texpr.ops": "ops", "texpr.ops.base": "op", "texpr.ops.elemwise": "elemwise",
        "texpr.ops.reductions": "reduce", "texpr.ops.linalg": "linalg", "texpr.ops.control": "control",
        "texpr.ops.conv": "conv", "texpr.ops.shaping": "shaping", "texpr.errors": "errors", "texpr.graph": "graph",
        "texpr.rewrites": "rewrite", "texpr.autodiff": "autodiff", "texpr.scan": "scan",
        "texpr.serialize": "serialize", "texpr.diagnostics": "diagnostics", "texpr.dtypes": "dtypes",
        "texpr.runtime": "vm", "texpr.shared": "shared",
    }
    sys.modules["texpr"] = P
    for name, m in mods.items():
        sys.modules[name] = _m(m)
    sys.modules["texpr.interp"] = _interp()
    sys.modules["texpr.alloc"] = _alloc()
    _testing()


install()
