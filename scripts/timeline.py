"""Per-CTA phase timeline of one GEMV (clock64 deltas from kernel entry).
usage: python scripts/timeline.py ROWS COLS"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200._native import check, lib  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
REP = int(sys.argv[3]) if len(sys.argv) > 3 else 1
layer = qw.synth_layer(rows, cols, seed=7)
dl = qw.DeviceLayer(layer)
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
y = torch.empty(rows, device="cuda")
E = lib().qw_debug_timeline_events()
grid = dl.info["quads"] if dl.info["quads"] < 148 else 148
names = ["entry", "dep resolved", "prologue done", "first unit in", "consumers done", "y written",
         "outliers done", "x landed", "x-indep done", "gathered", "-", "-"]
for trial in range(2):
    st = torch.zeros(grid * E, dtype=torch.int64, device="cuda")
    for _ in range(3):  # warm
        dl.matvec(x, out=y)
    check(lib().qw_debug_timeline(dl._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                  C.c_void_p(st.data_ptr()), REP, 0,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    if trial == 0:
        import oracle
        ref = oracle.matvec_f64(layer, x.cpu().numpy())
        yy = y.cpu().numpy()
        print("  rel-L2 after the diagnostic launch:", float(np.linalg.norm(yy - ref) / np.linalg.norm(ref)))
    a = st.cpu().numpy().reshape(grid, E).astype(np.int64)
    d = a - a[:, :1]
    print(f"trial {trial}: cycles from entry (mean / max over CTAs)")
    if REP > 1:
        nq = dl.info["quads"] / grid
        span = d[:, 4] - d[:, 2]
        print(f"  repeat {REP}: consumer loop {span.mean():.0f} cycles -> {span.mean() / (REP * nq):.1f} cycles/quad")
    for i in np.argsort(d.mean(0)):
        if d[:, i].max() <= 0 or d[:, i].min() < 0: continue
        print(f"  {names[i]:15s} {d[:, i].mean():9.0f} {d[:, i].max():9.0f}")
