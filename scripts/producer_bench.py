"""quantize_layer: the CPU producer (all host threads) vs the GPU producer
(qw_device_quantize), same inputs, outputs compared byte for byte (QWL1).
usage: python scripts/producer_bench.py [RxC ...]"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2311_16442_b200 as qw  # noqa: E402

shapes = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [(4096, 4096), (11008, 4096), (28672, 8192)]
tmp = Path(tempfile.mkdtemp())
qw.quantize_layer_gpu(qw.synth_gaussian(64, 256, 1), qw.synth_calibration(256, 1))  # warm the context
for rows, cols in shapes:
    w = qw.synth_gaussian(rows, cols, 7)
    h = qw.synth_calibration(cols, 7)
    t0 = time.perf_counter()
    cpu = qw.quantize_layer(w, h)
    t1 = time.perf_counter()
    gpu = qw.quantize_layer_gpu(w, h)
    t2 = time.perf_counter()
    qw.write_packed_layer(cpu, str(tmp / "c.qwl"))
    qw.write_packed_layer(gpu, str(tmp / "g.qwl"))
    same = (tmp / "c.qwl").read_bytes() == (tmp / "g.qwl").read_bytes()
    print(json.dumps({"shape": f"{rows}x{cols}", "cpu_s": round(t1 - t0, 3), "cpu_threads": os.cpu_count(),
                      "gpu_s": round(t2 - t1, 3), "speedup": round((t1 - t0) / (t2 - t1), 2),
                      "bit_identical": same}), flush=True)
