cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/timeline.py 4096 4096 2>&1 | tail -11
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 300 python scripts/chain_timing.py $s 64 | grep -v single; done
