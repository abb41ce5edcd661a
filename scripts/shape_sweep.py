"""BASELINE configs 1, 4 and 5 (N=1) on the batch-1 path: per-call time of a
dependent PDL chain of N distinct copies of one layer (inputs > L2), with the
parity of the first copy checked against the f64 oracle.
  config 1: q_proj 4096x4096, group2 128
  config 4: Llama-2-13B shapes (5120x5120, 13824x5120, 5120x13824), outlier ratio 0.1 .. 1 %
  config 5: Llama-2-70B shapes (8192x8192, 1024x8192, 28672x8192, 8192x28672) on one GPU
usage: python scripts/shape_sweep.py [N] [simt|mma]  -> one JSON line per case"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (checker only)
import paper_2311_16442_b200 as qw  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
KERNEL = sys.argv[2] if len(sys.argv) > 2 else "simt"
PEAK = 6554.2
cases = [("cfg1 q_proj g2=128", 4096, 4096, 128, 0.002)]
for r in (0.001, 0.002, 0.005, 0.01):
    cases += [(f"cfg4 13B qkvo r={r}", 5120, 5120, 16, r), (f"cfg4 13B gate/up r={r}", 13824, 5120, 16, r),
              (f"cfg4 13B down r={r}", 5120, 13824, 16, r)]
cases += [("cfg5 70B q/o", 8192, 8192, 16, 0.002), ("cfg5 70B k/v", 1024, 8192, 16, 0.002),
          ("cfg5 70B gate/up", 28672, 8192, 16, 0.002), ("cfg5 70B down", 8192, 28672, 16, 0.002)]
for name, rows, cols, g2, ratio in cases:
    layer = qw.synth_layer(rows, cols, seed=7, group2=g2, outlier_ratio=ratio)
    base = qw.DeviceLayer(layer, kernel=KERNEL)
    n = max(2, min(N, int(4 * 126e6 / qw.payload_bytes(layer)) + 1))
    dls = [base] + [base.clone() for _ in range(n - 1)]
    x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
    ys = torch.empty(n, rows, device="cuda")

    def run():
        for i, d in enumerate(dls):
            d.matvec(x, out=ys[i], pdl=True)
    run()
    torch.cuda.synchronize()
    ref = oracle.matvec_f64(layer, x.cpu().numpy())
    rel = float(np.linalg.norm(ys[0].cpu().numpy() - ref) / np.linalg.norm(ref))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    R = 10
    e0.record()
    for _ in range(R):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (R * n)
    balg = qw.payload_bytes(layer) + 4 * (rows + cols)
    print(json.dumps({"case": name, "kernel": KERNEL, "rows": rows, "cols": cols, "group2": g2, "outlier_ratio": ratio,
                      "nnz": int(layer.nnz),
                      "us_per_call": round(us, 3), "gb_s": round(balg / us / 1e3, 1),
                      "pct_of_hbm_peak": round(100 * balg / us / 1e3 / PEAK, 1), "rel_l2_vs_f64": rel,
                      "copies": n}), flush=True)

# GQA q/k/v of Llama-2-70B as ONE group launch (rows 8192 + 1024 + 1024)
layers = [qw.synth_layer(r, 8192, seed=30 + i) for i, r in enumerate((8192, 1024, 1024))]
n = 8
groups, outs = [], []
for c in range(n):
    dls = [qw.DeviceLayer(L, kernel=KERNEL) for L in layers]
    groups.append(qw.LayerGroup(dls))
    outs.append([torch.empty(L.cfg.rows, device="cuda") for L in layers])
x = torch.from_numpy(qw.synth_activation(8192, 8)).cuda()


def run_g():
    for g_, o in zip(groups, outs):
        g_.matvec(x, outs=o, pdl=True)
run_g()
torch.cuda.synchronize()
rel = max(float(np.linalg.norm(o.cpu().numpy() - oracle.matvec_f64(L, x.cpu().numpy())) /
                np.linalg.norm(oracle.matvec_f64(L, x.cpu().numpy()))) for L, o in zip(layers, outs[0]))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run_g()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (10 * n)
balg = sum(qw.payload_bytes(L) + 4 * (L.cfg.rows + L.cfg.cols) for L in layers)
print(json.dumps({"case": "cfg5 70B q/k/v GQA group launch", "kernel": KERNEL, "rows": 10240, "cols": 8192, "group2": 16,
                  "outlier_ratio": 0.002, "nnz": int(sum(L.nnz for L in layers)), "us_per_call": round(us, 3),
                  "gb_s": round(balg / us / 1e3, 1), "pct_of_hbm_peak": round(100 * balg / us / 1e3 / PEAK, 1),
                  "rel_l2_vs_f64": rel, "copies": n}), flush=True)
