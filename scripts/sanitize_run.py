"""Small invocations of every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the batch-1 kernels (K2 SIMT,
K2m warp MMA), column launches, the tcgen05 GEMM K4 with its x prologue
(cluster split-K and stream-K), a layer group, the dequant / unpack kernels
and the GPU producer.  Prints one line per step; the sanitizer's own summary
is the result.
usage: compute-sanitizer --tool memcheck python scripts/sanitize_run.py [step-name filter]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16442_b200 as qw  # noqa: E402


ONLY = sys.argv[1] if len(sys.argv) > 1 else ""


def step(name, fn):
    if ONLY not in name:
        return
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    for rows, cols, ratio in ((64, 512, 0.01), (1000, 2048, 0.005)):
        layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=ratio)
        xs = torch.from_numpy(np.stack([qw.synth_activation(cols, 40 + i) for i in range(16)])).cuda()
        for kernel in ("simt", "mma"):
            dl = qw.DeviceLayer(layer, kernel=kernel)
            step(f"{rows}x{cols} {kernel} batch 1", lambda: dl.matvec(xs[0].contiguous()))
            step(f"{rows}x{cols} {kernel} batch 1 pdl", lambda: dl.matvec(xs[0].contiguous(), pdl=True))
            step(f"{rows}x{cols} {kernel} columns b=3", lambda: dl.matvec(xs[:3].contiguous(), batched="columns"))
            step(f"{rows}x{cols} {kernel} columns b=11", lambda: dl.matvec(xs[:11].contiguous(), batched="columns"))
            dl.close()
        dl = qw.DeviceLayer(layer)
        for b in (2, 8, 16):
            step(f"{rows}x{cols} K4 b={b}", lambda: dl.matvec(xs[:b].contiguous(), batched="gemm", pdl=True))
        step(f"{rows}x{cols} reconstruct_dense", lambda: dl.reconstruct_dense())
        step(f"{rows}x{cols} unpack", lambda: dl.unpack())
        dl.close()
    # stream-K geometry (80 tiles x 4 weight stages over the SMs)
    layer = qw.synth_layer(10240, 2048, seed=3, outlier_ratio=0.002)
    dl = qw.DeviceLayer(layer)
    xs = torch.from_numpy(np.stack([qw.synth_activation(2048, 60 + i) for i in range(3)])).cuda()
    step("10240x2048 K4 stream-K b=3", lambda: dl.matvec(xs, batched="gemm"))
    dl.close()
    # a layer group (one launch for three layers sharing x)
    layers = [qw.DeviceLayer(qw.synth_layer(r, 1024, seed=r, outlier_ratio=0.005)) for r in (256, 128, 128)]
    grp = qw.LayerGroup(layers)
    x = torch.from_numpy(qw.synth_activation(1024, 5)).cuda()
    step("group of 3 batch 1", lambda: grp.matvec(x))
    step("group of 3 batch 4", lambda: grp.matvec(torch.stack([x] * 4).contiguous()))
    grp.close()
    # the GPU producer
    w = qw.synth_gaussian(96, 512, 9)
    h = qw.synth_calibration(512, 9)
    step("quantize_layer_gpu 96x512", lambda: qw.quantize_layer_gpu(w, h, outlier_ratio=0.01))
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
