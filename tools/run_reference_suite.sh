#!/bin/bash
# The reference's own test suite (pkg/tests/test_*.py, all seven files) against this
# package: `texpr` is aliased to paper_1605_02688_b200 by tests/refsuite/texpr_shim.py.
# baseline/_ref_tests is a git-ignored copy of /root/reference/pkg/tests made in
# the build container (cp /root/reference/pkg/tests/*.py baseline/_ref_tests/).
# Deselected tests and why: profiles/r02_reference_suite.md.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
T=baseline/_ref_tests
DESELECT=(
  # monkey-patch f.thunks[node.id] (per-node Python thunks; the VM replays a captured CUDA graph)
  --deselect $T/test_runtime.py::test_midway_injected_failure_keeps_shared
  --deselect $T/test_rewrites.py::test_transpose_executes_as_view
  # destroy_map marking by the `inplace` stage (replaced by the device planner's liveness reuse)
  --deselect $T/test_rewrites.py::test_inplace_marks_add_destroying_unused_input
  --deselect $T/test_rewrites.py::test_inplace_rejects_would_be_cycle
  --deselect $T/test_serialize.py::test_function_roundtrip_preserves_inplace_marks
  # creation tracebacks on variables (reference srcinfo.py: a debugging aid outside the hot path)
  --deselect $T/test_graph.py::test_creation_trace_recorded
)
PYTHONPATH=tests/refsuite:. timeout ${RTIMEOUT:-900} python -m pytest -p texpr_shim -p no:cacheprovider -q -rA \
  $T/test_ops.py $T/test_runtime.py $T/test_rewrites.py $T/test_autodiff.py $T/test_graph.py \
  $T/test_scan.py $T/test_serialize.py "${DESELECT[@]}" ${RPYARGS} > gpurun_out/refsuite.log 2>&1
echo "refsuite exit $?" >> gpurun_out/summary.txt
tail -n 5 gpurun_out/refsuite.log
