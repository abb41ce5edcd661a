cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/batch_sweep.py > gpurun_out/batch_sweep_v16.jsonl 2>/dev/null; tail -1 gpurun_out/batch_sweep_v16.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_k4_gate_stream python scripts/prof_batch.py 11008 4096 8 > gpurun_out/ncu_k4.out 2>&1; tail -2 gpurun_out/ncu_k4.out
