cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench $?" >> $O/summary.txt
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mlp.csv python tools/profile_run.py --only mlp --steps 2 > $O/prof_mlp.log 2>&1
cat $O/summary.txt
