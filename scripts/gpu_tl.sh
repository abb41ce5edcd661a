cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in 1 2; do timeout 600 python -m pytest tests -m gpu -q --timeout 120 2>&1 | grep -E "passed|failed|Warning" | tail -2; done
