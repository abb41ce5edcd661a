import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2311_16442_b200 as qw
rows, cols, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
base = qw.DeviceLayer(qw.synth_layer(rows, cols, seed=7))
dls = [base] + [base.clone() for _ in range(n - 1)]
grp = qw.LayerGroup(dls)
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
for _ in range(4):
    grp.matvec(x)
torch.cuda.synchronize()
print("ok")
