cd $GRAFT_REPO_ROOT; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/timeline.py 4096 4096 1 2>&1 | tail -22
timeout 300 python scripts/timeline.py 4096 4096 20 2>&1 | grep repeat
timeout 300 python scripts/timeline.py 4096 11008 20 2>&1 | grep repeat
