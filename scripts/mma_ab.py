"""A/B of the batch-1 kernels on single layers: tensor-core K2m (default)
vs the SIMT K2 (DeviceLayer(kernel=...)).  Per-call µs of a CUDA graph of
N distinct copies (inputs > L2), dependent (PDL chain) and independent.
usage: python scripts/mma_ab.py [shape ...]  (shape = ROWSxCOLS)"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [
    (4096, 4096), (11008, 4096), (4096, 11008), (28672, 8192), (1024, 8192)]
PEAK = 6554.2
for rows, cols in shapes:
    layer = qw.synth_layer(rows, cols, seed=7)
    balg = qw.payload_bytes(layer) + 4 * (rows + cols)
    n = max(4, min(32, int(4 * 126e6 / balg) + 1))
    out = {"shape": f"{rows}x{cols}", "copies": n}
    for mode in ("mma", "simt"):
        base = qw.DeviceLayer(layer, kernel=mode)
        dls = [base] + [base.clone() for _ in range(n - 1)]
        x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
        ys = torch.empty(n, rows, device="cuda")
        for dep in (True, False):
            def run():
                for i, d in enumerate(dls):
                    d.matvec(x, out=ys[i], pdl=True, x_independent=not dep)
            run()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                run()
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            R = 20
            e0.record()
            for _ in range(R):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (R * n)
            out[f"{mode}_{'dep' if dep else 'ind'}_us"] = round(us, 3)
            out[f"{mode}_{'dep' if dep else 'ind'}_pct"] = round(100 * balg / us / 1e3 / PEAK, 1)
        del dls, base
    print(json.dumps(out), flush=True)
