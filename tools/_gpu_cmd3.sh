cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
timeout 1200 python -m pytest tests -q -m "gpu and slow" -x > $O/tests_slow.log 2>&1; echo "tests_slow $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/summary.txt
cat $O/summary.txt
