cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for sh in G8 G7 G2 G1; do python tools/gemm_ab.py $sh TX_GEMM_NO3D=1 >> $O/ab.log 2>&1; done
for sh in G1 G2 G6; do python tools/gemm_ab.py $sh TX_GEMM_NO_TMA_STORE=1 >> $O/ab.log 2>&1; done
python tools/gemm_ab.py G7 TX_GEMM_BN=192 >> $O/ab.log 2>&1
python tools/gemm_ab.py G8 TX_GEMM_CG=1 >> $O/ab.log 2>&1
cat $O/ab.log
