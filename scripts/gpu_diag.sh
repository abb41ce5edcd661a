cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/timeline.py 4096 4096 1 2>&1 | tail -40
timeout 300 python scripts/timeline.py 4096 4096 20 2>&1 | grep repeat
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 300 python scripts/chain_timing.py $s 64; done
