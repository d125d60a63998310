cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_device_ops.py tests/test_device_configs.py tests/test_device_serialize.py -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
timeout 300 python tools/gemm_bench.py > $O/gemm.log 2>&1
TX_GEMM_NO_TMA_AUX=1 timeout 300 python tools/gemm_bench.py G6 > $O/gemm_noaux.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench $?" >> $O/summary.txt
cat $O/summary.txt; tail -n 3 $O/tests.log; cut -c1-100 $O/gemm.log $O/gemm_noaux.log
