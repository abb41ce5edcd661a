cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "batch" 2>&1 | tail -2
timeout 600 python scripts/batch_sweep.py > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err
python - <<'P'
import json
for l in open("gpurun_out/batch_sweep.jsonl"):
    d = json.loads(l); print(d["shape"], d["batch"], d["us_per_call"], d["gb_s"])
P
