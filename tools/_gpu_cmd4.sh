cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for g in G1 G8; do
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o $O/full_$g python tools/gemm_bench.py $g > $O/ncu_$g.log 2>&1
done
TX_GEMM_CG=1 timeout 300 python tools/gemm_bench.py G1 G8 > $O/gemm_cg1.log 2>&1
timeout 300 python tools/gemm_bench.py G1 G8 > $O/gemm_cg2.log 2>&1
cat $O/gemm_cg1.log $O/gemm_cg2.log
