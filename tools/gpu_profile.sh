#!/bin/bash
# ncu evidence: launch list of every kernel (cold-cache, serialised) and one
# full-set capture of the top kernels.  Numbers printed under ncu are never bench values.
cd "${GRAFT_REPO_ROOT:-$(pwd)}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/profile_run.py --steps 2 > gpurun_out/prof_run.log 2>&1
echo "launches exit $?" >> gpurun_out/summary.txt
for spec in ${FULL:-"ew:tx_ew_flat:1" "mlp:tc_gemm:2"}; do
  IFS=: read only kern skip <<< "$spec"
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
    -o gpurun_out/full_${only} python tools/profile_run.py --only $only --steps 2 > gpurun_out/full_${only}.log 2>&1
  echo "full $only exit $?" >> gpurun_out/summary.txt
done
