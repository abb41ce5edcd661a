"""Run the matvec of one synthetic layer a few times (for ncu captures).
usage: python scripts/prof_one.py ROWS COLS [reps] [outlier_ratio] [kernel]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ratio = float(sys.argv[4]) if len(sys.argv) > 4 else 0.002
kernel = sys.argv[5] if len(sys.argv) > 5 else "auto"
layer = qw.synth_layer(rows, cols, seed=7, outlier_ratio=ratio)
dl = qw.DeviceLayer(layer, kernel=kernel)
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
y = torch.empty(rows, device="cuda")
for _ in range(reps):
    dl.matvec(x, out=y)
torch.cuda.synchronize()
print("ok", rows, cols, "K2m" if dl.uses_tensor_core else "K2", float(y.abs().sum()))
