"""Small invocations of every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): the batch-1 kernels (K2 SIMT,
K2m warp MMA), column launches, the tcgen05 GEMM K4 with its x prologue
(cluster split-K and stream-K), a layer group, the dequant / unpack kernels,
the persistent chain kernel, the fused TP exchange (push / wait / reduce)
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


def peer_exchange():
    """qw_matvec_push (GEMV epilogue stores into both ranks' buffers and
    counts arrivals) + qw_peer_wait + qw_peer_reduce, ranks as streams (every
    push enqueued before any wait)."""
    import ctypes as C

    from paper_2311_16442_b200._native import check, lib
    from paper_2311_16442_b200.tp import shard_layer
    layer = qw.synth_layer(512, 1024, seed=8, outlier_ratio=0.005)
    x = torch.from_numpy(qw.synth_activation(1024, 8)).cuda()
    world, dls, ranges = 2, [], None
    for r in range(world):
        shard, ranges_r, _ = shard_layer(layer, r, world, "col")
        ranges = ranges_r or ranges
        dls.append(qw.DeviceLayer(shard, 0, kernel="simt"))
    bufs = [torch.zeros(512, device="cuda") for _ in range(world)]
    flags = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    y_loc = [torch.zeros(d.rows, device="cuda") for d in dls]
    out = torch.zeros(512, device="cuda")
    expected = sum(int(lib().qw_push_arrivals(d._h)) for d in dls)
    streams = [torch.cuda.Stream() for _ in range(world)]
    torch.cuda.synchronize()

    def run():
        for r in range(world):
            peer_y = (C.c_void_p * world)(*[b.data_ptr() + 4 * ranges[r][0] for b in bufs])
            peer_f = (C.c_void_p * world)(*[f.data_ptr() for f in flags])
            check(lib().qw_matvec_push(dls[r]._h, C.c_void_p(x.data_ptr()), C.c_void_p(y_loc[r].data_ptr()),
                                       peer_y, peer_f, world, C.c_void_p(streams[r].cuda_stream), 0))
        for r in range(world):
            check(lib().qw_peer_wait(C.c_void_p(flags[r].data_ptr()), expected, C.c_void_p(streams[r].cuda_stream)))
        check(lib().qw_peer_reduce(C.c_void_p(bufs[0].data_ptr()), 1, 512, C.c_void_p(out.data_ptr()),
                                   C.c_void_p(streams[0].cuda_stream)))
    step("peer exchange 2 ranks", run)


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
    # a wide layer at group2 = 1 (a 2-order row per row): K2's plan needs
    # three CTAs per SM (run in waves)
    layer = qw.synth_layer(1200, 13792, seed=5, group2=1, outlier_ratio=0.005)
    dl = qw.DeviceLayer(layer, kernel="simt")
    xw = torch.from_numpy(qw.synth_activation(13792, 5)).cuda()
    step("1200x13792 g2=1 K2 (several CTAs per SM)", lambda: dl.matvec(xw))
    dl.close()
    # a layer group (one launch for three layers sharing x)
    layers = [qw.DeviceLayer(qw.synth_layer(r, 1024, seed=r, outlier_ratio=0.005)) for r in (256, 128, 128)]
    grp = qw.LayerGroup(layers)
    x = torch.from_numpy(qw.synth_activation(1024, 5)).cuda()
    step("group of 3 batch 1", lambda: grp.matvec(x))
    step("group of 3 batch 4", lambda: grp.matvec(torch.stack([x] * 4).contiguous()))
    grp.close()
    # the persistent chain kernel: two dependent steps
    sq = qw.DeviceLayer(qw.synth_layer(512, 512, seed=4, outlier_ratio=0.01))
    x0 = torch.from_numpy(qw.synth_activation(512, 6)).cuda()
    y1, y2 = torch.empty(512, device="cuda"), torch.empty(512, device="cuda")
    chain = qw.DecodeChain([([sq], x0, [y1], False), ([sq], y1, [y2], True)])
    step("chain kernel 2 steps", lambda: chain.run())
    chain.close()
    # the fused TP exchange: 2 ranks as streams of this process, column split
    peer_exchange()
    # the GPU producer
    w = qw.synth_gaussian(96, 512, 9)
    h = qw.synth_calibration(512, 9)
    step("quantize_layer_gpu 96x512", lambda: qw.quantize_layer_gpu(w, h, outlier_ratio=0.01))
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
