cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 1 2 3; do echo "QW_CTAS_PER_SM=$c"; QW_CTAS_PER_SM=$c timeout 300 python scripts/timeline.py 4096 4096 20 2>&1 | grep repeat | head -1; for s in "4096 4096" "11008 4096"; do QW_CTAS_PER_SM=$c timeout 300 python scripts/chain_timing.py $s 64 | grep "distinct"; done; done
