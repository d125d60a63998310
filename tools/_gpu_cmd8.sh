cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/summary.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench $?" >> $O/summary.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "bench_ref $?" >> $O/summary.txt
for w in mlp logreg; do
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv python tools/profile_run.py --only $w --steps 2 > $O/prof_$w.log 2>&1
done
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:tx_ew_flat -s 1 -c 1 -o $O/full_ew python tools/profile_run.py --only ew --steps 2 > $O/full_ew.log 2>&1
cat $O/summary.txt; tail -n 2 $O/bench_ref.log
