#!/bin/bash
# One GPU session: build check, device tests (each bounded), smoke, bench.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for t in ${TESTS:-test_device_runtime test_device_ops test_device_configs}; do
  timeout ${TTIMEOUT:-400} python -m pytest tests/$t.py -q -m "gpu and not slow" --durations=5 ${PYARGS} > gpurun_out/$t.log 2>&1
  echo "$t exit $?" >> gpurun_out/summary.txt
done
if [ -n "$SMOKE" ]; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/summary.txt; fi
if [ -n "$BENCH" ]; then timeout ${BTIMEOUT:-900} python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/summary.txt; fi
for f in gpurun_out/*.log; do echo "== $f"; tail -n 3 "$f"; done
