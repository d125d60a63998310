cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_device_scan.py -q -m gpu -x > $O/scan.log 2>&1; echo "scan $?" >> $O/summary.txt
timeout 900 python -m pytest tests -q -m "gpu and not slow" > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
cat $O/summary.txt; tail -n 40 $O/scan.log; tail -n 5 $O/tests.log
