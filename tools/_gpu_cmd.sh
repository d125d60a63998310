cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_device_ops.py tests/test_device_configs.py -q -m "gpu and not slow" -x > $O/tests.log 2>&1; echo "tests $?" >> $O/summary.txt
timeout 300 python tools/gemm_bench.py > $O/gemm.log 2>&1; echo "gemm $?" >> $O/summary.txt
for g in G2 G6 G7; do
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $O/full_$g python tools/gemm_bench.py $g > $O/ncu_$g.log 2>&1
done
for w in mlp logreg; do
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$w.csv python tools/profile_run.py --only $w --steps 2 > $O/prof_$w.log 2>&1
done
python tools/e2e_probe.py > $O/probe.log 2>&1
cat $O/summary.txt
