cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_torch_ops.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "torch or straight or batched or a_tile or smoke" > gpurun_out/g3_pytest.txt 2>&1; tail -15 gpurun_out/g3_pytest.txt
timeout 900 python scripts/batch_sweep.py 16 > gpurun_out/g3_batch.jsonl 2>&1; python - <<'PY'
import json
for l in open("gpurun_out/g3_batch.jsonl"):
    try: d=json.loads(l)
    except Exception: print(l[:150]); continue
    print(d["shape"], d["batch"], d["mode"], d["us_per_call"], d["gb_s"], d["path"])
PY
