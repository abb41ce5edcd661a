cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py > gpurun_out/batch_sweep_v17.jsonl 2>/dev/null
QW_DEBUG_KNOBS=1 QW_GEMM_NOSTREAM=1 timeout 600 python scripts/batch_sweep.py 24 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['batch'] > 1 and d['shape']=='gate_proj': print('nostream', d['shape'], d['batch'], d['us_per_call'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k4_gate_stream_v17 python scripts/prof_batch.py 11008 4096 8 > gpurun_out/ncu_k4.out 2>&1; tail -1 gpurun_out/ncu_k4.out
