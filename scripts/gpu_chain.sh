cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 300 python scripts/chain_timeline.py 4096 4096 12 | tail -5
timeout 300 python scripts/chain_timeline.py 11008 4096 8 | tail -3
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 300 python scripts/chain_timing.py $s 32 | grep distinct; done
