cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 0 1; do echo "QW_NO_PRE=$v"; QW_NO_PRE=$v timeout 300 python scripts/chain_timeline.py 4096 4096 12 | tail -4; done
echo "independent"; timeout 300 python scripts/chain_timeline.py 4096 4096 12 --indep | tail -4
timeout 300 python scripts/chain_timeline.py 11008 4096 8 --indep | tail -3
