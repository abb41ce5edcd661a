cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] in (2,16): print(d['shape'], d['batch'], d['us_per_call'])"
echo "== skip xprep (timing only)"
QW_SKIP_XPREP=1 timeout 600 python scripts/batch_sweep.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] in (2,16): print(d['shape'], d['batch'], d['us_per_call'])"
