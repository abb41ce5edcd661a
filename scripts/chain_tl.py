"""Per-step phase timeline of the tensor-core decode-chain kernel.
usage: QW_DEBUG_KNOBS=1 QW_DEBUG_MMA_TL=1 python scripts/chain_tl.py [decoder_layers] [indep]
Prints, per step kind (q/k/v, o, gate/up, down), the median over CTAs and
steps of each phase (µs): dependency wait, x staging + B build, items, CSR
meet, reduction, release; and the step period."""
import ctypes as C
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_16442_b200 as qw  # noqa: E402
from paper_2311_16442_b200._native import lib  # noqa: E402
from paper_2311_16442_b200.stack import LinearStack  # noqa: E402

assert os.environ.get("QW_DEBUG_MMA_TL") == "1" and os.environ.get("QW_DEBUG_KNOBS") == "1", \
    "set QW_DEBUG_KNOBS=1 QW_DEBUG_MMA_TL=1"
NL = int(sys.argv[1]) if len(sys.argv) > 1 else 4
indep = len(sys.argv) > 2 and sys.argv[2] == "indep"
cache = Path(os.environ.get("QW_BENCH_CACHE", Path(tempfile.gettempdir()) / "qw_bench_cache"))
cache.mkdir(parents=True, exist_ok=True)
base = bench.make_layers(0, 1, cache, os.cpu_count() or 1)
dls = [qw.DeviceLayer(L, 0, kernel="mma") for L in base]
per = []
for l in range(NL):
    for i, d in enumerate(dls):
        per.append(d if l == 0 else d.clone())
groups = []
for l in range(NL):
    b = 7 * l
    groups += [[b, b + 1, b + 2], [b + 3], [b + 4, b + 5], [b + 6]]
st = LinearStack(per, device=0, batch=1, pdl=True, groups=groups)
x = np.concatenate([qw.synth_activation(L.cfg.cols, 5) for _ in range(NL) for L in base])
st.x.copy_(torch.from_numpy(x))
ch = st.make_chain([not indep and gi > 0 for gi in range(len(st.groups))])
for _ in range(5):
    ch.run()
torch.cuda.synchronize()
n = len(st.groups)
grid = 148
buf = (C.c_ulonglong * (n * grid * 8))()
rc = lib().qw_debug_chain_timeline(ch._h, buf, n * grid * 8)
assert rc == 0, rc
t = np.frombuffer(buf, dtype=np.uint64).reshape(n, grid, 8).astype(np.int64)
t0 = t[:, :, 0].min()
kinds = ["qkv", "o", "gateup", "down"]
names = ["dep_wait", "x+B", "items", "csr_meet", "reduce", "release"]
print(f"{NL} decoder layers, {'independent' if indep else 'dependent'}; total {(t[-1,:,6].max()-t0)/1e3:.1f} us")
for k in range(4):
    rows = t[k::4]
    ph = np.stack([rows[:, :, 4] - rows[:, :, 0], rows[:, :, 1] - rows[:, :, 4], rows[:, :, 2] - rows[:, :, 1],
                   rows[:, :, 3] - rows[:, :, 2], rows[:, :, 5] - rows[:, :, 3], rows[:, :, 6] - rows[:, :, 5]], -1)
    med = np.median(ph.reshape(-1, 6), 0) / 1e3
    mx = np.median(ph.max(1), 0) / 1e3
    # step period: max over CTAs of release - min start
    period = np.median((rows[:, :, 6].max(1) - rows[:, :, 0].min(1))) / 1e3
    prod = np.median((rows[:, :, 7] - rows[:, :, 0]).reshape(-1)) / 1e3
    print(f"{kinds[k]:7s} period {period:6.2f} | " + " ".join(f"{nm} {m:5.2f}/{x:5.2f}" for nm, m, x in zip(names, med, mx)) +
          f" | producer last issue {prod:6.2f}")
