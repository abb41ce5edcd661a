cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "chain or group" 2>&1 | tail -2
python scripts/prof_chain.py 8 5; python scripts/prof_chain.py 8 5 indep
