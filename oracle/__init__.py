"""CPU oracle for the texpr compiled-graph hot path — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference's per-op host kernels
(``/root/reference/pkg/src/texpr/ops/*.py`` perform methods) and of its
plain interpreter (``interp.py:20-51``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it,
and only as the checker / the timed CPU reference — the product package never
imports it, and there is no CPU fallback in the product.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(importable in the build container) on seeded inputs and stores the results in
``tests/golden/texpr_goldens.npz``; ``tests/test_oracle.py`` checks this
restatement against those vectors (bit-exact: same NumPy calls, same order).
"""
