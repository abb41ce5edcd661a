cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "QW_NPRE_MAX=0" "QW_NPRE_MAX=4" "QW_NPRE_MAX=2" "QW_NPRE_MAX=4 QW_XGATE=6"; do
  env $v timeout 600 python bench.py --no-cpu --steps 10 > gpurun_out/b.json 2> gpurun_out/b.err
  echo "$v: $(python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['value'],d['independent']['value'],d['roofline']['achieved'])" 2>&1 | tail -1)"
done
