set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_list.out 2>&1
tail -3 gpurun_out/ncu_list.out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -c 7 -o gpurun_out/prof_gemv python bench.py --layers 1 --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_full.out 2>&1
tail -3 gpurun_out/ncu_full.out
ls -la gpurun_out
