cd $GRAFT_REPO_ROOT
O=gpurun_out/$RUN; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/dump_rowfuse.py > $O/rowfuse_logreg.cu 2>&1
python tools/overhead_probe.py > $O/overhead.log 2>&1
echo done
