cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/b.json 2> gpurun_out/b.err; tail -c 700 gpurun_out/b.json
timeout 600 python bench.py --compare-chain --no-cpu --steps 5 > gpurun_out/b2.json 2> gpurun_out/b2.err
python -c "import json;d=json.load(open('gpurun_out/b2.json'));print(d['value'],d['chain_kernel'])"
