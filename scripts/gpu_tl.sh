cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['clocks'])"
