"""Per-launch time of chains of GEMVs under different conditions (diagnostic).
usage: python scripts/chain_timing.py ROWS COLS [N]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 64
layer = qw.synth_layer(rows, cols, seed=7)
base = qw.DeviceLayer(layer)
distinct = [base] + [base.clone() for _ in range(N - 1)]
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
ys = torch.empty(N, rows, device="cuda")
ws = qw.Workspace(0, cols + 64, 1)
bytes_per = qw.payload_bytes(layer) + 4 * (rows + cols)


def graph_of(layers, pdl):
    def run():
        for i, dl in enumerate(layers):
            dl.matvec(x, out=ys[i], workspace=ws, pdl=pdl)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    return g


def t_graph(g, reps=20):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us per graph


for name, layers in (("distinct", distinct), ("same(L2-hot)", [base] * N)):
    for pdl in (True, False):
        us = t_graph(graph_of(layers, pdl)) / N
        print(f"{rows}x{cols} {name:13s} pdl={pdl!s:5s}: {us:7.3f} us/launch  "
              f"{bytes_per / us / 1e3:8.1f} GB/s")
# single cold launch
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
distinct[-1].matvec(x, out=ys[0], workspace=ws)
e1.record()
torch.cuda.synchronize()
print(f"single launch (events): {e0.elapsed_time(e1) * 1e3:.2f} us")
