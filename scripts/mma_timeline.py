"""Global-clock timeline of the decode chain (q/k/v group, o, gate/up group,
down) x L decoder layers on K2m (warp-MMA) group launches, CUDA graph + PDL
(diagnostic; the K2 version is step_timeline.py).
usage: python scripts/mma_timeline.py [L] [simt]"""
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
bases = [qw.DeviceLayer(qw.synth_layer(r, c, seed=7 + i), kernel="mma") for i, (r, c, n) in enumerate(shapes)]
launches = []
for l in range(L):
    for i, (r, c, n) in enumerate(shapes):
        dls = [bases[i].clone() for _ in range(n)]
        grp = qw.LayerGroup(dls)
        x = torch.from_numpy(qw.synth_activation(c, 8)).cuda()
        ys = [torch.empty(r, device="cuda") for _ in range(n)]
        launches.append((names[i], grp, dls, x, ys))
E = lib().qw_debug_timeline_events()
G = 448
st = torch.zeros(len(launches), G * E, dtype=torch.int64, device="cuda")


def run():
    s = torch.cuda.current_stream().cuda_stream
    for k, (nm, grp, dls, x, ys) in enumerate(launches):
        ptrs = (C.c_void_p * len(ys))(*[y.data_ptr() for y in ys])
        check(lib().qw_debug_group_timeline(grp._h, C.c_void_p(x.data_ptr()), ptrs, C.c_void_p(st[k].data_ptr()), 1,
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
ev = {"entry": 0, "copies": 7, "csr_req": 8, "dep": 10, "x": 1, "B": 11, "items": 2, "csr": 6, "met": 3,
      "sums": 9, "end": 5}
print("per launch: median / max over CTAs (us from the previous launch's last end stamp)")
print("launch   " + " ".join(f"{k:>12s}" for k in ev))
prev = None
for k, (nm, *_rest) in enumerate(launches):
    r = a[k]
    r = r[r[:, 0] > 0] - t0
    if prev is None:
        prev = r[:, 0].min()
    cols = []
    for name, e in ev.items():
        v = r[:, e]
        v = v[v > -t0]
        cols.append(f"{(np.median(v) - prev) / 1e3:5.2f}/{(v.max() - prev) / 1e3:5.2f}" if v.size else "   -/-   ")
    print(f"{nm:8s} " + " ".join(f"{c:>12s}" for c in cols))
    prev = r[:, 5].max()
