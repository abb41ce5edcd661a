cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for ks in 1 2 3 4; do echo "== ks $ks"; QW_GEMM_KS=$ks timeout 600 python scripts/batch_sweep.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] in (4,16): print(d['shape'], d['batch'], d['us_per_call'])"; done
