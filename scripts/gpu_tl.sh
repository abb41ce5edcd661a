cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mode in pdl nopdl pdl; do echo "== $mode"
timeout 600 python scripts/batch_sweep.py 24 $mode 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], d['batch'], d['us_per_call'])"; done
