cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
echo "== L=1 watch"; QW_CHAIN_WATCH=1 timeout 120 python scripts/_dbg_hang2.py 1 2>&1 | tail -2
echo "== L=1"; timeout 120 python scripts/_dbg_hang2.py 1 2>&1 | tail -1
echo "== L=2"; timeout 120 python scripts/_dbg_hang2.py 2 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -1
timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['independent']['value'],d['chain_kernel']['value'],d['roofline']['achieved'])"
