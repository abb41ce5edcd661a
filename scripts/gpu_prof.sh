cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/prof_q python scripts/prof_one.py 4096 4096 3 > gpurun_out/prof_q.out 2>&1
tail -2 gpurun_out/prof_q.out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/prof_down python scripts/prof_one.py 4096 11008 3 > gpurun_out/prof_down.out 2>&1
tail -2 gpurun_out/prof_down.out
