cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/g2_pytest.txt 2>&1; tail -25 gpurun_out/g2_pytest.txt
timeout 600 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err; tail -c 2500 gpurun_out/g2_bench.json; tail -2 gpurun_out/g2_bench.err
