"""Where the GPU matvec departs from the f64 oracle (diagnostic).
usage: python scripts/debug_parity.py ROWS COLS [ratio]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import oracle
import paper_2311_16442_b200 as qw
rows, cols = int(sys.argv[1]), int(sys.argv[2])
ratio = float(sys.argv[3]) if len(sys.argv) > 3 else 0.002
layer = qw.synth_layer(rows, cols, seed=7, outlier_ratio=ratio)
x = qw.synth_activation(cols, 8)
dl = qw.DeviceLayer(layer)
y = dl.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
ref = oracle.matvec_f64(layer, x)
rel = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
err = np.abs(y - ref)
bad = np.where(err > 1e-2 * np.abs(ref).max())[0]
print(rows, cols, "rel", rel, "nbad", bad.size, "first", bad[:20], "quads", bad[:20] // 4)
if bad.size:
    q = bad // 4
    print("bad quad range", q.min(), q.max(), "per-CTA quads", dl.info["quads"] / 148)
    for r in bad[:5]:
        print("  row", r, y[r], ref[r])
