# ncu full capture of one repeat-mode GEMV (consumers re-run resident quads: compute-rate profile)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:gemv_kernel -s 3 -c 1 -o gpurun_out/prof_rep python scripts/timeline.py 4096 4096 20 > gpurun_out/prof_rep.out 2>&1
tail -1 gpurun_out/prof_rep.out
