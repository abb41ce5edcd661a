cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_nccl.py -m gpu -q > gpurun_out/p1_tpnccl.txt 2>&1; tail -3 gpurun_out/p1_tpnccl.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/p1_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/p1_bench_under_ncu.log 2>&1; tail -2 gpurun_out/p1_bench_under_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 3 -c 1 -o gpurun_out/p1_gemv_group python scripts/prof_group.py 4096 4096 3 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/p1_gemv_group.ncu-rep > gpurun_out/p1_gemv_group_sum.txt 2>&1; head -20 gpurun_out/p1_gemv_group_sum.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mma_gemv -s 2 -c 1 -o gpurun_out/p1_mma_13b_down python scripts/prof_one.py 5120 13824 3 0.01 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/p1_mma_13b_down.ncu-rep > gpurun_out/p1_mma_13b_down_sum.txt 2>&1; head -20 gpurun_out/p1_mma_13b_down_sum.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o gpurun_out/p1_simt_13b_down python scripts/prof_one.py 5120 13824 3 0.01 simt > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/p1_simt_13b_down.ncu-rep > gpurun_out/p1_simt_13b_down_sum.txt 2>&1; head -20 gpurun_out/p1_simt_13b_down_sum.txt
