cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m "gpu and not slow" > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
cat $O/summary.txt; grep -E "FAIL|Error|passed|failed" $O/tests.log | head -20
