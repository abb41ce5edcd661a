import sys
sys.path.insert(0, '.')
import numpy as np, torch
import oracle
import paper_2311_16442_b200 as qw
rows, cols, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
layer = qw.synth_layer(rows, cols, seed=7)
base = qw.DeviceLayer(layer)
dls = [base] + [base.clone() for _ in range(n - 1)]
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
ref = torch.from_numpy(oracle.matvec_f64(layer, x.cpu().numpy()).astype(np.float32)).cuda()
tol = 1e-2 * ref.abs().max()
bad_total, bad_runs = 0, 0
for r in range(reps):
    ys = torch.zeros(n, rows, device="cuda")
    for i, d in enumerate(dls):
        d.matvec(x, out=ys[i], pdl=False)
    torch.cuda.synchronize()
    nb = int(((ys - ref).abs() > tol).sum())
    bad_total += nb
    bad_runs += nb > 0
print(f"{rows}x{cols} copies {n} reps {reps}: runs with bad rows {bad_runs}, bad rows {bad_total}")
