"""Global-clock timeline of a PDL chain of distinct GEMVs (diagnostic).
usage: python scripts/chain_timeline.py ROWS COLS [N]
Per kernel: first CTA entry, last 'prologue done', last consumer done, last y
written (ns, relative to the first kernel's first entry)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200._native import check, lib  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
N = int(sys.argv[3]) if len(sys.argv) > 3 else 12
FLAGS = 3 | (4 if '--indep' in sys.argv else 0)
layer = qw.synth_layer(rows, cols, seed=7)
base = qw.DeviceLayer(layer)
dls = [base] + [base.clone() for _ in range(N - 1)]
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
ys = torch.empty(N, rows, device="cuda")
E = lib().qw_debug_timeline_events()
G = 448
st = torch.zeros(N, G * E, dtype=torch.int64, device="cuda")
def launch_all():
    s = torch.cuda.current_stream().cuda_stream
    for i, dl in enumerate(dls):
        check(lib().qw_debug_timeline(dl._h, C.c_void_p(x.data_ptr()), C.c_void_p(ys[i].data_ptr()),
                                      C.c_void_p(st[i].data_ptr()), 1, FLAGS, C.c_void_p(s)))


launch_all()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    launch_all()
for trial in range(3):
    g.replay()
torch.cuda.synchronize()
a = st.cpu().numpy().reshape(N, G, E).astype(np.int64)
grid = int((a[0, :, 0] > 0).sum())
a = a[:, :grid, :]
t0 = a[0, :, 0].min()
print(f"{rows}x{cols}, {N} kernels, grid {grid}: ns from first entry")
print("   k   entry0  entry_max   pre_max   dep_min   dep_max    x_max  gath_max  prolog_max  unit0_max  cons_max    y_max   y_span")
prev = None
for i in range(N):
    r = a[i] - t0
    line = (f"  {i:2d} {r[:, 0].min():8d} {r[:, 0].max():9d} {r[:, 8].max():9d} {r[:, 1].min():9d} {r[:, 1].max():9d} {r[:, 7].max():8d} {r[:, 9].max():9d} {r[:, 2].max():10d} {r[:, 3].max():10d} "
            f"{r[:, 4].max():9d} {r[:, 5].max():8d} {r[:, 5].max() - r[:, 0].min():8d}")
    print(line)
ends = [(a[i, :, 5] - t0).max() for i in range(N)]
print("per-kernel step (y_max deltas, ns):", np.diff(ends)[2:].mean().round(1))
