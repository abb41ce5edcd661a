cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['independent']['value'],d['chain_kernel']['value'],d['roofline']['achieved'])"
timeout 1200 python scripts/shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep.err
python - <<'P'
import json
for l in open("gpurun_out/shape_sweep.jsonl"):
    d = json.loads(l); print(d["case"], d["us_per_call"], d["gb_s"], d["pct_of_hbm_peak"], "%.1e" % d["rel_l2_vs_f64"])
P
timeout 600 python scripts/batch_sweep.py > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err; tail -2 gpurun_out/batch_sweep.err
