# scratch iteration on a B200: parity of the batch-1 paths, then the bench (MMA default vs SIMT)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${TAG:-it}
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q ${PYARGS} > gpurun_out/${T}_pytest.txt 2>&1
tail -15 gpurun_out/${T}_pytest.txt
timeout 300 python bench.py --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
QW_DEBUG_SIMT=1 timeout 300 python bench.py --no-cpu > gpurun_out/${T}_bench_simt.json 2>> gpurun_out/${T}_bench.err
python - <<'PY'
import json,os
T=os.environ.get("TAG","it")
for f in (f"gpurun_out/{T}_bench.json", f"gpurun_out/{T}_bench_simt.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"], d["independent"]["value"], d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e)
PY
tail -5 gpurun_out/${T}_bench.err
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mma_gemv -s 3 -c 1 -o gpurun_out/${T}_mma_group python scripts/prof_group.py 4096 4096 3 > gpurun_out/${T}_ncu.out 2>&1
  python scripts/ncu_summary.py gpurun_out/${T}_mma_group.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1
  head -60 gpurun_out/${T}_ncu_summary.txt
fi
