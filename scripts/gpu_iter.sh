# iteration loop: build, smoke, GPU parity, short bench, ncu of the q_proj GEMV
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/prof_q python scripts/prof_one.py 4096 4096 3 > gpurun_out/prof_q.out 2>&1
tail -1 gpurun_out/prof_q.out
