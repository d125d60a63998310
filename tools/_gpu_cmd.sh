cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/summary.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench $?" >> $O/summary.txt
TX_REDUCE_NO_TMA=1 timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_notma.log 2>&1; echo "bench_notma $?" >> $O/summary.txt
for w in mlp logreg reduce; do
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv python tools/profile_run.py --only $w --steps 2 > $O/prof_$w.log 2>&1
done
cat $O/summary.txt
