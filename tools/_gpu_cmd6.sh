cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
timeout 600 python tools/lstm_bench.py small > $O/lstm.log 2>&1; echo "lstm small $?" >> $O/summary.txt
timeout 600 python tools/lstm_bench.py medium >> $O/lstm.log 2>&1; echo "lstm medium $?" >> $O/summary.txt
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lstm.csv python tools/lstm_bench.py small --steps 1 > $O/lstm_ncu.log 2>&1
cat $O/summary.txt; tail -n 5 $O/tests.log; tail -n 30 $O/lstm.log
