cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 300 python scripts/chain_timing.py $s 64; done
