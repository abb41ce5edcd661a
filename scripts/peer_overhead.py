"""Cost of the fused peer exchange on one GPU: a 4096x4096 layer as a
one-rank column split -- qw_matvec_push into its own buffer + qw_peer_wait --
against the plain matvec, in CUDA-graph chains of distinct copies.
usage: python scripts/peer_overhead.py [rows cols]"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200._native import check, lib  # noqa: E402

rows, cols = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4096, 4096)
N = 24
base = qw.DeviceLayer(qw.synth_layer(rows, cols, seed=7), kernel="simt")
dls = [base] + [base.clone() for _ in range(N - 1)]
x = torch.from_numpy(qw.synth_activation(cols, 8)).cuda()
ys = torch.empty(N, rows, device="cuda")
full = torch.empty(N, rows, device="cuda")
flags = torch.zeros(N, dtype=torch.int32, device="cuda")
arr = int(lib().qw_push_arrivals(base._h))


def plain():
    for i, d in enumerate(dls):
        d.matvec(x, out=ys[i], pdl=True)


def pushed():
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for i, d in enumerate(dls):
        py = (C.c_void_p * 1)(full[i].data_ptr())
        pf = (C.c_void_p * 1)(flags[i:i + 1].data_ptr())
        check(lib().qw_matvec_push(d._h, C.c_void_p(x.data_ptr()), C.c_void_p(ys[i].data_ptr()), py, pf, 1, s, 1))
        check(lib().qw_peer_wait(C.c_void_p(flags[i:i + 1].data_ptr()), arr, s))


out = {"shape": f"{rows}x{cols}"}
for name, fn in (("plain", plain), ("push_wait", pushed)):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    out[f"{name}_us"] = round(e0.elapsed_time(e1) * 1e3 / (20 * N), 3)
assert torch.equal(full, ys)
print(json.dumps(out))
