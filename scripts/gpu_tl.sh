cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batched" 2>&1 | tail -2
L=paper_2311_16442_b200/lib/libqweight_b200.so
for v in old new newstream; do echo "== $v"
if [ $v = newstream ]; then cp abtmp/new.so $L; unset QW_GEMM_NOSTREAM; else cp abtmp/$v.so $L; export QW_GEMM_NOSTREAM=1; fi
timeout 600 python scripts/batch_sweep.py 24 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] in (2,8,16): print(d['shape'], d['batch'], d['us_per_call'])"; done
