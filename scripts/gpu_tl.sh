cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batched" 2>&1 | tail -2
timeout 600 python scripts/batch_sweep.py 24 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] > 1: print(d['shape'], d['batch'], d['us_per_call'])"
