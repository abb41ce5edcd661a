# full round check: build, smoke, gpu tests, bench (+reference arm), launch list,
# ncu full captures of the GEMV group kernels, the chain kernel and the K4 GEMM
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --launch chain --no-cpu > gpurun_out/bench_chain.json 2> gpurun_out/bench_chain.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_list.out 2>&1; tail -1 gpurun_out/ncu_list.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -c 4 -o gpurun_out/prof_gemv python scripts/step_timeline.py 1 > gpurun_out/ncu_full.out 2>&1; tail -1 gpurun_out/ncu_full.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/prof_chain python scripts/prof_chain.py 1 1 > gpurun_out/ncu_chain.out 2>&1; tail -1 gpurun_out/ncu_chain.out
timeout 600 python scripts/batch_sweep.py > gpurun_out/batch_sweep.jsonl 2> gpurun_out/batch_sweep.err; tail -3 gpurun_out/batch_sweep.jsonl
timeout 1200 python scripts/shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep.err; tail -3 gpurun_out/shape_sweep.jsonl
ls -la gpurun_out | head -40
