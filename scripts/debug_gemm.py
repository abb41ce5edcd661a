"""One small batched matvec through K4 (debug)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import oracle
import paper_2311_16442_b200 as qw
rows, cols, batch = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (96, 512, 2)))
layer = qw.synth_layer(rows, cols, seed=5)
dl = qw.DeviceLayer(layer)
print("launches", dl.launches_per_matvec(batch), flush=True)
xs = np.stack([qw.synth_activation(cols, 300 + b) for b in range(batch)])
Y = dl.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
for b in range(batch):
    ref = oracle.matvec_f64(layer, xs[b])
    print(b, "rel", float(np.linalg.norm(Y[b] - ref) / np.linalg.norm(ref)), Y[b][:4], ref[:4])
