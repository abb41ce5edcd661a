cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in simt mma; do timeout 900 python scripts/shape_sweep.py 16 $k > gpurun_out/s1_sweep_$k.jsonl 2>&1; done
python - <<'PY'
import json
rows={}
for k in ("simt","mma"):
    for l in open(f"gpurun_out/s1_sweep_{k}.jsonl"):
        try: d=json.loads(l)
        except Exception: print(l[:200]); continue
        rows.setdefault(d["case"],{})[k]=d
for c,v in rows.items():
    print(f"{c:32s} simt {v.get('simt',{}).get('us_per_call','-'):>8} us {v.get('simt',{}).get('pct_of_hbm_peak','-'):>5}%  mma {v.get('mma',{}).get('us_per_call','-'):>8} us {v.get('mma',{}).get('pct_of_hbm_peak','-'):>5}%  relL2 {v.get('simt',{}).get('rel_l2_vs_f64',0):.1e}/{v.get('mma',{}).get('rel_l2_vs_f64',0):.1e}")
PY
