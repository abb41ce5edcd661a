"""Per-CTA %globaltimer phases of one K4 batched matvec (ns from the first setup stamp)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2311_16442_b200 as qw
from paper_2311_16442_b200._native import check, lib
rows, cols, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
layer = qw.synth_layer(rows, cols, seed=7)
dl = qw.DeviceLayer(layer)
xs = torch.from_numpy(np.stack([qw.synth_activation(cols, 50 + i) for i in range(b)])).cuda()
y = torch.empty(b, rows, device="cuda")
st = torch.zeros(512 * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    st.zero_()
    check(lib().qw_debug_gemm_timeline(dl._h, C.c_void_p(xs.data_ptr()), b, C.c_void_p(y.data_ptr()),
                                       C.c_void_p(st.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
a = st.cpu().numpy().reshape(512, 8)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = ["setup", "s3 W present", "CTA joined", "cluster joined", "prologue done", "sums done (t0)", "y stored", "acc ready"]
print(f"{rows}x{cols} b={b}: {a.shape[0]} CTAs")
for i, nm in enumerate(names):
    v = a[:, i]
    v = v[v > 0] - t0
    if v.size:
        print(f"  {nm:11s} min {v.min():8d} mean {v.mean():10.0f} max {v.max():8d}")
