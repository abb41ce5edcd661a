"""BASELINE config 3: Llama-2-7B shapes, batch 1/2/3/4/8/16: the batched
policy against both forced paths (K4 tcgen05 GEMM; the batch-1 kernel over
the columns, up to 8 columns per launch).  Per-call time from a CUDA-graph
chain of N distinct layer copies (inputs > L2).  With QW_DEBUG_KNOBS=1
QW_COLUMN_GROUP=0 the column path runs one launch per column (A/B).
usage: python scripts/batch_sweep.py [N] [nopdl] [simt|mma|auto]  -> one JSON line per (shape, batch, path)"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 24
PDL = not (len(sys.argv) > 2 and sys.argv[2] == "nopdl")
KERNEL = sys.argv[3] if len(sys.argv) > 3 else "auto"
GROUPED = os.environ.get("QW_COLUMN_GROUP", "1") != "0" or os.environ.get("QW_DEBUG_KNOBS") != "1"
for name, rows, cols in (("q_proj", 4096, 4096), ("gate_proj", 11008, 4096), ("down_proj", 4096, 11008)):
    layer = qw.synth_layer(rows, cols, seed=7)
    base = qw.DeviceLayer(layer, kernel=KERNEL)
    dls = [base] + [base.clone() for _ in range(N - 1)]
    payload = qw.payload_bytes(layer)
    for b, mode in [(1, "auto")] + [(b, m) for b in (2, 3, 4, 5, 6, 7, 8, 16) for m in ("auto", "gemm", "columns")]:
        xs = torch.from_numpy(np.stack([qw.synth_activation(cols, 50 + i) for i in range(b)])).cuda()
        ys = torch.empty(N, b, rows, device="cuda")

        def run():
            for i, d in enumerate(dls):
                d.matvec(xs, out=ys[i], pdl=PDL, batched=mode)
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        R = 10
        for _ in range(R):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (R * N)
        balg = payload + 4 * b * (rows + cols)
        launches = base.launches_per_matvec(b, mode)
        gemm = base.batched_path(b, mode) == "gemm" if b > 1 else False
        kern = "K2m" if base.uses_tensor_core else "K2"
        path = ("K4 tcgen05 GEMM" if gemm else
                f"{kern} over {b} column(s), {launches} launch(es)" if GROUPED else f"{b} x batch-1 {kern}")
        line = {"shape": name, "rows": rows, "cols": cols, "batch": b, "us_per_call": round(us, 3),
                "gb_s": round(balg / us / 1e3, 1), "tflops": round(2 * b * rows * cols / us / 1e6, 2),
                "mode": mode, "launches": launches, "kernel": kern, "grouped_columns": GROUPED, "path": path}
        print(json.dumps(line), flush=True)
