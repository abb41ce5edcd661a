"""Global-clock timeline of a grouped decode chain (q/k/v group, o, gate/up
group, down) x L decoder layers, CUDA graph + PDL (diagnostic).
usage: python scripts/step_timeline.py [L] [pf]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200._native import check, lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
shapes = [(4096, 4096, 3), (4096, 4096, 1), (11008, 4096, 2), (4096, 11008, 1)]
names = ["qkv", "o", "gate_up", "down"]
bases = [qw.DeviceLayer(qw.synth_layer(r, c, seed=7 + i)) for i, (r, c, n) in enumerate(shapes)]
launches = []
for l in range(L):
    for i, (r, c, n) in enumerate(shapes):
        dls = [bases[i].clone() for _ in range(n)]
        grp = qw.LayerGroup(dls)
        x = torch.from_numpy(qw.synth_activation(c, 8)).cuda()
        ys = [torch.empty(r, device="cuda") for _ in range(n)]
        launches.append((names[i], grp, dls, x, ys))
if len(sys.argv) > 2 and sys.argv[2] == "pf":  # each launch prefetches the next one's weights into L2
    for k, (nm, grp, dls, x, ys) in enumerate(launches):
        grp.set_prefetch(launches[(k + 1) % len(launches)][2])
E = lib().qw_debug_timeline_events()
G = 448
st = torch.zeros(len(launches), G * E, dtype=torch.int64, device="cuda")


def run():
    s = torch.cuda.current_stream().cuda_stream
    for k, (nm, grp, dls, x, ys) in enumerate(launches):
        ptrs = (C.c_void_p * len(ys))(*[y.data_ptr() for y in ys])
        check(lib().qw_debug_group_timeline(grp._h, C.c_void_p(x.data_ptr()), ptrs, C.c_void_p(st[k].data_ptr()), 3,
                                            C.c_void_p(s)))


run()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    run()
for _ in range(3):
    st.zero_()
    g.replay()
torch.cuda.synchronize()
a = st.cpu().numpy().reshape(len(launches), G, E).astype(np.int64)
t0 = a[0, :, 0][a[0, :, 0] > 0].min()
ev = {"entry": 0, "dep": 1, "xind": 8, "x": 7, "gath": 9, "prolog": 2, "cons": 4, "csr": 6, "y": 5}
print("per launch: median / max over CTAs (us from the previous launch's last y store)")
print("launch   " + " ".join(f"{k:>12s}" for k in ev))
prev_y = None
for k, (nm, *_rest) in enumerate(launches):
    r = a[k]
    r = r[r[:, 0] > 0] - t0
    if prev_y is None:
        prev_y = r[:, 0].min()
    cols = []
    for name, e in ev.items():
        v = r[:, e]
        v = v[v > -t0]
        cols.append(f"{(np.median(v) - prev_y) / 1e3:5.2f}/{(v.max() - prev_y) / 1e3:5.2f}")
    print(f"{nm:8s} " + " ".join(f"{c:>12s}" for c in cols))
    prev_y = r[:, 5].max()
