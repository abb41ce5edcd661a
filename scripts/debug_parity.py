"""Print where the GPU matvec departs from the f64 oracle for a few small layers."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import oracle
import paper_2311_16442_b200 as qw
for rows, cols in [(64, 512), (20, 80), (8, 64)]:
    layer = qw.synth_layer(rows, cols, seed=rows * 31 + cols)
    x = qw.synth_activation(cols, rows + 100)
    dl = qw.DeviceLayer(layer)
    y = dl.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = oracle.matvec_f64(layer, x)
    bad = np.where(~np.isclose(y, ref, rtol=1e-2, atol=1e-2 * np.abs(ref).max()))[0]
    print(rows, cols, "bad rows", bad[:40], "n", bad.size)
    for r in bad[:6]:
        print("   row", r, y[r], ref[r])
