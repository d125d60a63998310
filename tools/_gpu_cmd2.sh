cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_device_runtime.py tests/test_device_configs.py -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
python tools/overhead_probe.py > $O/overhead.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench $?" >> $O/summary.txt
cat $O/summary.txt
