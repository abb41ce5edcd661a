"""Print where the GPU matvec departs from the f64 oracle for a few layers
(rows, cols, group2, outlier ratio), diagnostic."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import oracle
import paper_2311_16442_b200 as qw
CASES = [(64, 512, 16, 0.01, 0.25), (16, 1024, 16, 0.0, 0.25), (16, 1024, 16, 0.0, 0.0), (16, 1024, 16, 0.0, 1.0),
         (16, 512, 16, 0.0, 0.0), (16, 512, 16, 0.0, 1.0), (16, 768, 16, 0.0, 0.0), (16, 2048, 16, 0.0, 0.0)]
for rows, cols, g2, ratio, alpha in CASES:
    layer = qw.synth_layer(rows, cols, seed=rows * 31 + cols, group2=g2, outlier_ratio=ratio, alpha=alpha)
    x = qw.synth_activation(cols, rows + 100)
    dl = qw.DeviceLayer(layer)
    y = dl.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = oracle.matvec_f64(layer, x)
    bad = np.where(~np.isclose(y, ref, rtol=1e-2, atol=1e-2 * np.abs(ref).max()))[0]
    print(rows, cols, g2, ratio, alpha, "bad rows", bad[:40], "n", bad.size, "nan", np.isnan(y).sum())
    for r in bad[:2]:
        print("   row", r, y[r], ref[r])
