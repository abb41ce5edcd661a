cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k4 python scripts/prof_batch.py 4096 4096 16 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k4_gate python scripts/prof_batch.py 11008 4096 16 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
