# scratch iteration script: GPU parity + a short bench (edited per experiment)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1
timeout 600 python bench.py --no-cpu > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['independent']['value'],d['roofline']['achieved'],d['e2e']['value'])"
