# iteration loop: build, smoke, GPU parity, timeline, chain timing, repeat-mode ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/timeline.py 4096 4096 1 2>&1 | tail -8
timeout 300 python scripts/timeline.py 4096 4096 20 2>&1 | grep repeat
for s in "4096 4096" "11008 4096" "4096 11008"; do timeout 300 python scripts/chain_timing.py $s 64 | grep "distinct"; done
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:gemv_kernel -s 3 -c 1 -o gpurun_out/prof_rep python scripts/timeline.py 4096 4096 20 > gpurun_out/prof_rep.out 2>&1
tail -1 gpurun_out/prof_rep.out
