import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2311_16442_b200 as qw
rows, cols, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
layer = qw.synth_layer(rows, cols, seed=7)
dl = qw.DeviceLayer(layer)
xs = torch.from_numpy(np.stack([qw.synth_activation(cols, 50 + i) for i in range(b)])).cuda()
for _ in range(3):
    y = dl.matvec(xs)
torch.cuda.synchronize()
print("ok")
