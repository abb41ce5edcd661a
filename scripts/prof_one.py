"""Run the matvec of one synthetic layer a few times (for ncu captures).
usage: python scripts/prof_one.py ROWS COLS [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
layer = qw.synth_layer(rows, cols, seed=7)
dl = qw.DeviceLayer(layer)
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
y = torch.empty(rows, device="cuda")
for _ in range(reps):
    dl.matvec(x, out=y)
torch.cuda.synchronize()
print("ok", rows, cols, float(y.abs().sum()))
