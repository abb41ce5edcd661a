"""Run the persistent decode-chain kernel over L Llama-2-7B decoder layers
(grouped steps: q/k/v, o, gate/up, down), for ncu captures and timing.
usage: python scripts/prof_chain.py [L] [reps] [indep]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
indep = len(sys.argv) > 3 and sys.argv[3] == "indep"
shapes = [(4096, 4096, 3), (4096, 4096, 1), (11008, 4096, 2), (4096, 11008, 1)]
bases = [qw.DeviceLayer(qw.synth_layer(r, c, seed=7 + i)) for i, (r, c, n) in enumerate(shapes)]
steps, nbytes = [], 0
for l in range(L):
    for i, (r, c, n) in enumerate(shapes):
        dls = [bases[i].clone() for _ in range(n)]
        x = torch.from_numpy(qw.synth_activation(c, 8)).cuda()
        ys = [torch.empty(r, device="cuda") for _ in range(n)]
        steps.append((dls, x, ys, not indep and len(steps) > 0))
        nbytes += n * (dls[0].info["payload_bytes"] + 4 * (r + c))
ch = qw.DecodeChain(steps)
for _ in range(2):
    ch.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ch.run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"chain L={L} {'indep' if indep else 'dep'}: {ms * 1e3 / L:.2f} us/decoder layer, {nbytes / ms / 1e6:.1f} GB/s")
