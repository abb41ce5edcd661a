"""GPU parity: the sm_100a path against the C oracle (and through it the
reference) on identical inputs.

  * K0 unpack and K1 dequant are bit-exact (reference unpack_layer /
    reconstruct_dense), pads and outlier slots included.
  * K2+K3 matvec y matches matvec_reference_f64 within the north-star
    tolerance: rel-L2 <= 1e-2 and max-abs <= 1e-2 * max|y| (fp16 partial
    sums; typically ~5e-4).
Edge cases follow the reference tests: tails (T2 != T4), pads, pure 2-bit /
pure 4-bit layers, rows not a multiple of 4, odd group2, zero x, no
outliers, dense outliers, random zero2 (helpers.hpp random_groups).
"""
import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _torch():
    import torch
    return torch


def rel_l2(y, ref):
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(np.asarray(y, np.float64) - ref) / (den if den else 1.0))


KERNELS = ["simt", "mma"]  # K2 (SIMT) and K2m (warp MMA) batch-1 kernels


def check_layer(layer, x, device=0, kernel="simt"):
    torch = _torch()
    dl = qw.DeviceLayer(layer, device, kernel=kernel)
    # K1: bit-exact reconstruct_dense
    w = dl.reconstruct_dense().cpu().numpy()
    ref_w = oracle.reconstruct_dense(layer)
    assert np.array_equal(w.view(np.uint32), ref_w.view(np.uint32))
    # K0: bit-exact unpack_layer
    got = {k: v.cpu().numpy() for k, v in dl.unpack().items()}
    ref = oracle.unpack(layer)
    for k in ref:
        assert np.array_equal(got[k], ref[k]), k
    # K2/K3: y within tolerance of the f64 oracle
    y = dl.matvec(torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()
    ref_y = oracle.matvec_f64(layer, x)
    assert np.all(np.isfinite(y))
    err = rel_l2(y, ref_y)
    assert err <= TOL, err
    scale = np.max(np.abs(ref_y)) if ref_y.size else 0.0
    assert np.max(np.abs(y - ref_y)) <= TOL * max(scale, 1e-30) + 1e-30
    return err, dl


GEOMS = [
    # rows, cols, alpha, group2, ratio
    (20, 80, 0.25, 16, 0.002),     # pads + tails (test_engine.cpp:51-60)
    (24, 160, 0.5, 16, 0.005),     # tail4-heavy
    (9, 96, 0.0, 16, 0.0),         # pure 2-bit, rows % 4 != 0
    (9, 96, 1.0, 16, 0.0),         # pure 4-bit
    (37, 160, 0.25, 16, 0.01),     # odd rows, dense outliers
    (64, 512, 0.25, 5, 0.01),      # group2 not a multiple of 4
    (130, 1024, 0.25, 128, 0.002), # g2 = 128 (config 1 "group 128")
    (16, 1024, 0.25, 16, 0.0),     # zero outliers (test_engine.cpp:71-76)
    (40, 512, 0.25, 1, 0.01),      # group2 = 1: every row its own 2-order block
    (21, 768, 0.25, 3, 0.01),      # group2 = 3
    (64, 28672, 0.25, 16, 0.002),  # 70B down width: 56 chunks, 4 per warp
]


def test_too_wide_layer_for_the_simt_kernel():
    """80 chunks of 32 groups exceed the SIMT kernel's 60: forcing it is a
    clean QW_ERR_UNSUPPORTED, and the default upload serves the layer with the
    tensor-core kernel K2m, within the tolerance of the oracle."""
    torch = _torch()
    layer = qw.synth_layer(16, 40960, seed=3, alpha=0.25, group2=16, outlier_ratio=0.002)
    with pytest.raises(qw.QWeightError) as ei:
        qw.DeviceLayer(layer, kernel="simt")
    assert ei.value.status == 5
    dl = qw.DeviceLayer(layer)
    assert dl.uses_tensor_core
    x = qw.synth_activation(40960, 4)
    y = dl.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_l2(y, oracle.matvec_f64(layer, x)) <= TOL


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("rows,cols,alpha,g2,ratio", GEOMS)
def test_geometries(rows, cols, alpha, g2, ratio, kernel):
    layer = qw.synth_layer(rows, cols, seed=rows * 31 + cols, alpha=alpha, group2=g2,
                           outlier_ratio=ratio)
    x = qw.synth_activation(cols, rows + 100)
    check_layer(layer, x, kernel=kernel)


def test_zero_activation_gives_zero():
    torch = _torch()
    layer = qw.synth_layer(12, 64, seed=10)
    dl = qw.DeviceLayer(layer)
    y = dl.matvec(torch.zeros(64, device="cuda")).cpu().numpy()
    assert np.all(y == 0.0)


@pytest.mark.parametrize("kernel", KERNELS)
def test_random_groups_with_nonzero_zero2(kernel):
    """helpers.hpp random_groups: random codes, zero2 0..15, fp16 scales."""
    rng = np.random.default_rng(5)
    base = qw.synth_layer(32, 256, seed=3)
    c = base.cfg
    layer = qw.PackedLayer(
        cfg=c, plan_bits=base.plan_bits, plan_perm=base.plan_perm,
        main=rng.integers(0, 256, base.main.size, dtype=np.uint8),
        tail2=rng.integers(0, 256, base.tail2.size, dtype=np.uint8),
        tail4=rng.integers(0, 256, base.tail4.size, dtype=np.uint8),
        secondary=rng.integers(0, 256, base.secondary.size, dtype=np.uint8),
        meta=rng.integers(0, 65536, base.meta.size, dtype=np.uint16),
        sorder_zero2=rng.integers(0, 16, base.sorder_zero2.size, dtype=np.uint8),
        # moderate scales keep the fp16 products finite
        sorder_scale2=np.array([qw_f16(v) for v in rng.uniform(0.01, 0.2, base.sorder_zero2.size)],
                               np.uint16),
        fourbit_scale=np.array([qw_f16(v) for v in rng.uniform(0.01, 0.5, base.fourbit_zero.size)],
                               np.uint16),
        fourbit_zero=rng.integers(0, 16, base.fourbit_zero.size, dtype=np.uint8),
        row_ptr=base.row_ptr, col_ind=base.col_ind, values=base.values)
    qw.validate_layer(layer)
    x = qw.synth_activation(256, 4)
    check_layer(layer, x, kernel=kernel)


def qw_f16(v: float) -> int:
    return int(np.float16(v).view(np.uint16))


@pytest.mark.parametrize("kernel", KERNELS)
def test_large_activation_range(kernel):
    """Power-of-two group scaling keeps fp16 partials finite for large x."""
    layer = qw.synth_layer(64, 512, seed=21)
    x = qw.synth_activation(512, 22) * np.float32(3e4)
    x[5] = 1e9
    err, _ = check_layer(layer, x, kernel=kernel)
    assert err < 5e-3


def test_batched_columns_match_single():
    torch = _torch()
    layer = qw.synth_layer(96, 512, seed=8)
    dl = qw.DeviceLayer(layer)
    xs = np.stack([qw.synth_activation(512, 50 + b) for b in range(4)])
    Y = dl.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
    for b in range(4):
        ref = oracle.matvec_f64(layer, xs[b])
        assert rel_l2(Y[b], ref) <= TOL


def test_checked_host_path_validates_activation():
    layer = qw.synth_layer(8, 64, seed=11)
    dl = qw.DeviceLayer(layer)
    with pytest.raises(qw.QWeightError):
        dl.matvec_checked(np.zeros(63, np.float32))
    bad = np.ones(64, np.float32)
    bad[7] = np.nan
    with pytest.raises(qw.QWeightError):
        dl.matvec_checked(bad)
    res = dl.matvec_checked(qw.synth_activation(64, 3))
    assert rel_l2(res.y, oracle.matvec_f64(layer, qw.synth_activation(64, 3))) <= TOL
    assert res.wall_ns > 0


def test_deterministic_runs():
    torch = _torch()
    layer = qw.synth_layer(128, 1024, seed=25)
    dl = qw.DeviceLayer(layer)
    x = torch.from_numpy(qw.synth_activation(1024, 26)).cuda()
    a = dl.matvec(x).cpu().numpy()
    b = dl.matvec(x).cpu().numpy()
    assert np.array_equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("rows,cols", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_llama7b_shapes(rows, cols, kernel):
    """Config 2 shapes at full size: bit-exact dequant + y tolerance."""
    layer = qw.synth_layer(rows, cols, seed=7)
    x = qw.synth_activation(cols, 8)
    err, _ = check_layer(layer, x, kernel=kernel)
    assert err < 2e-3


# ---------------------------------------------------------------- K4 (batched)
BATCH_GEOMS = [
    # rows, cols, batch: tensor-core path (paired tiles, group2 % 4 == 0)
    (96, 512, 2),       # one partial M tile
    (300, 1024, 5),     # 3 tiles, last partial; rows % 4 == 0
    (130, 768, 16),     # rows % 4 != 0 inside the last tile, full batch
    (512, 4096, 8),     # K split across CTAs (split-K fixup)
    (4096, 4096, 16),   # Llama-2-7B q_proj, batch 16
    (10240, 2048, 3),   # stream-K: 80 tiles x 4 weight stages over 148 CTAs (two-tile ranges)
    (11008, 4096, 4),   # Llama-2-7B gate_proj: stream-K, 86 tiles
    (8192, 8192, 8),    # Llama-2-70B q_proj: stream-K, 64 tiles x 16 weight stages
    (11008, 4096, 16),  # gate_proj, stream-K at the full batch
    (4096, 11008, 2),   # Llama-2-7B down_proj: cluster split-K, 86 sub-stages
]


@pytest.mark.parametrize("rows,cols,batch", BATCH_GEOMS)
def test_batched_tensor_core_path(rows, cols, batch):
    torch = _torch()
    layer = qw.synth_layer(rows, cols, seed=rows + cols + batch, outlier_ratio=0.005)
    dl = qw.DeviceLayer(layer)
    assert dl.launches_per_matvec(batch, "gemm") == 2, "expected x prologue + tcgen05 GEMM"
    # the default policy: K4 from 6 columns, the batch-1 kernel 8 columns to
    # a launch below
    min_b = 6
    assert dl.batched_path(batch) == ("gemm" if batch >= min_b else "columns")
    assert dl.launches_per_matvec(batch) == (2 if batch >= min_b else (batch + 7) // 8)
    xs = np.stack([qw.synth_activation(cols, 300 + b) for b in range(batch)])
    Y = dl.matvec(torch.from_numpy(xs).cuda(), batched="gemm").cpu().numpy()
    assert np.all(np.isfinite(Y))
    for b in range(batch):
        ref = oracle.matvec_f64(layer, xs[b])
        err = rel_l2(Y[b], ref)
        assert err <= TOL, (b, err)
        assert np.max(np.abs(Y[b] - ref)) <= TOL * np.max(np.abs(ref))
    # deterministic run to run (fixed split-K summation order)
    Y2 = dl.matvec(torch.from_numpy(xs).cuda(), batched="gemm").cpu().numpy()
    assert np.array_equal(Y, Y2)
    # the per-column path agrees within the tolerance
    Yc = dl.matvec(torch.from_numpy(xs).cuda(), batched="columns").cpu().numpy()
    for b in range(batch):
        assert rel_l2(Yc[b], oracle.matvec_f64(layer, xs[b])) <= TOL


@pytest.mark.parametrize("n,batch", [(2048, 2), (2048, 8), (4096, 16)])
def test_k4_dependent_chain_with_pdl(n, batch):
    """K4 calls whose x is the previous call's y, on ONE layer (the x
    prologue's scratch is reused by every call), launched back to back with
    programmatic dependent launch -- the prologue grid resident under the
    previous GEMM and reading the layer constants before its dependency wait
    (a plain launch above kPrepPdlMaxBlocks = 192 CTAs: the 4096 x 16 case):
    bit-identical to the same calls synchronised one by one, eager and as a
    replayed CUDA graph."""
    torch = _torch()
    layer = qw.synth_layer(n, n, seed=n + batch, outlier_ratio=0.005)
    dl = qw.DeviceLayer(layer)
    X = torch.from_numpy(np.stack([qw.synth_activation(n, 900 + b) for b in range(batch)])).cuda()
    steps = 6
    ref = [X]
    for _ in range(steps):
        ref.append(dl.matvec(ref[-1], batched="gemm", pdl=True))
        torch.cuda.synchronize()
    assert all(bool(torch.isfinite(r).all()) for r in ref)
    ys = [torch.empty(batch, n, device="cuda") for _ in range(steps)]

    def run():
        prev = X
        for i in range(steps):
            dl.matvec(prev, out=ys[i], batched="gemm", pdl=True)
            prev = ys[i]
    run()
    torch.cuda.synchronize()
    for i in range(steps):
        assert torch.equal(ys[i], ref[i + 1]), i
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    for _ in range(3):
        for y in ys:
            y.zero_()
        g.replay()
        torch.cuda.synchronize()
        for i in range(steps):
            assert torch.equal(ys[i], ref[i + 1]), i


COLUMN_GEOMS = [
    (96, 512, 0.01),      # one chunk, a few CTAs per column
    (1000, 4096, 0.005),  # rows not a multiple of 16 / 4
    (512, 11008, 0.01),   # K2m: three chunks (per-column chunk-partial slots)
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("rows,cols,ratio", COLUMN_GEOMS)
def test_column_launches_match_single_columns(rows, cols, ratio, kernel):
    """A batch on the batch-1 kernel: up to 8 columns share one launch (the
    grid split over the columns like a layer group).  Every column equals its
    own batch-1 launch bit for bit and the oracle within the tolerance."""
    torch = _torch()
    layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=ratio)
    dl = qw.DeviceLayer(layer, kernel=kernel)
    for batch in (2, 3, 5, 8, 11):
        assert dl.launches_per_matvec(batch, "columns") == (batch + 7) // 8
        xs = np.stack([qw.synth_activation(cols, 70 + b) for b in range(batch)])
        X = torch.from_numpy(xs).cuda()
        Y = dl.matvec(X, batched="columns").cpu().numpy()
        Y2 = dl.matvec(X, batched="columns").cpu().numpy()
        assert np.array_equal(Y, Y2)  # deterministic
        for b in range(batch):
            y1 = dl.matvec(X[b].contiguous()).cpu().numpy()
            assert np.array_equal(Y[b].view(np.uint32), y1.view(np.uint32)), (batch, b)
            ref = oracle.matvec_f64(layer, xs[b])
            assert rel_l2(Y[b], ref) <= TOL


def test_batched_unsupported_geometry_falls_back_to_columns():
    """Unpaired tiles (T2 != T4) keep the per-column fused GEMV (still exact semantics)."""
    torch = _torch()
    layer = qw.synth_layer(24, 160, seed=4, alpha=0.5)
    dl = qw.DeviceLayer(layer)
    assert dl.batched_path(3, "gemm") == "columns"
    assert dl.launches_per_matvec(3, "gemm") == 1  # three columns, one launch
    xs = np.stack([qw.synth_activation(160, 40 + b) for b in range(3)])
    Y = dl.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
    for b in range(3):
        assert rel_l2(Y[b], oracle.matvec_f64(layer, xs[b])) <= TOL


# ---------------------------------------------------------------- TP (1 rank over NCCL)
@pytest.mark.parametrize("mode", ["col", "row"])
def test_tp_linear_single_rank_nccl(mode):
    """The TP shard + NCCL collective path on one GPU (world size 1): the
    GPU code path end to end; multi-rank semantics are tested with gloo."""
    import os
    import torch.distributed as dist
    torch = _torch()
    from paper_2311_16442_b200.tp import TPLinear
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    layer = qw.synth_layer(256, 1024, seed=9, outlier_ratio=0.005)
    x = qw.synth_activation(1024, 10)
    try:
        tp = TPLinear(layer, 0, 1, mode, device="cuda:0")
        assert tp.device == torch.device("cuda", 0)
        y = tp.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel_l2(y, oracle.matvec_f64(layer, x)) <= TOL
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- group launch
@pytest.mark.parametrize("kernel", KERNELS)
def test_group_launch_matches_single_layers(kernel):
    """q/k/v-style group: three layers, one input, one fused launch; each
    output equals (bitwise) the single-layer launch and the f64 oracle."""
    torch = _torch()
    layers = [qw.synth_layer(512, 1024, seed=60 + i, outlier_ratio=0.005) for i in range(3)]
    dls = [qw.DeviceLayer(L, kernel=kernel) for L in layers]
    grp = qw.LayerGroup(dls)
    x = qw.synth_activation(1024, 61)
    xd = torch.from_numpy(x).cuda()
    outs = grp.matvec(xd)
    for L, d, o in zip(layers, dls, outs):
        y = o.cpu().numpy()
        assert rel_l2(y, oracle.matvec_f64(L, x)) <= TOL
        single = d.matvec(xd).cpu().numpy()
        assert rel_l2(y, single) <= 1e-6


@pytest.mark.parametrize("kernel", KERNELS)
def test_group_batch_launch_matches_single_columns(kernel):
    """A batched group launch (qw_group_matvec_batch: up to 8 / n columns of
    every layer in one grid) equals each layer's batch-1 launch per column,
    bit for bit; GQA-style unequal rows, n = 3 and n = 2."""
    torch = _torch()
    for rows, b_list in (((512, 128, 128), (2, 3, 5)), ((1024, 1024), (2, 4, 7))):
        layers = [qw.synth_layer(r, 2048, seed=90 + i + r, outlier_ratio=0.005) for i, r in enumerate(rows)]
        dls = [qw.DeviceLayer(L, kernel=kernel) for L in layers]
        grp = qw.LayerGroup(dls)
        for b in b_list:
            xs = np.stack([qw.synth_activation(2048, 91 + k) for k in range(b)])
            X = torch.from_numpy(xs).cuda()
            outs = grp.matvec(X)
            for L, d, o in zip(layers, dls, outs):
                assert o.shape == (b, d.rows)
                for k in range(b):
                    single = d.matvec(X[k].contiguous()).cpu().numpy()
                    assert np.array_equal(o[k].cpu().numpy().view(np.uint32), single.view(np.uint32)), (b, k)
                    assert rel_l2(o[k].cpu().numpy(), oracle.matvec_f64(L, xs[k])) <= TOL


def test_group_rejects_mismatched_geometry():
    a = qw.DeviceLayer(qw.synth_layer(64, 512, seed=1))
    b = qw.DeviceLayer(qw.synth_layer(64, 1024, seed=2))
    with pytest.raises(qw.QWeightError):
        qw.LayerGroup([a, b])


def test_prefetch_hint_leaves_results_unchanged():
    """qw_*_set_prefetch: a launch that also streams the next launch's weights
    into L2 computes bitwise the same outputs."""
    torch = _torch()
    la, lb = qw.synth_layer(512, 1024, seed=70), qw.synth_layer(256, 1024, seed=71)
    a, b = qw.DeviceLayer(la), qw.DeviceLayer(lb)
    grp = qw.LayerGroup([qw.DeviceLayer(qw.synth_layer(512, 1024, seed=72 + i)) for i in range(2)])
    xd = torch.from_numpy(qw.synth_activation(1024, 73)).cuda()
    ya, yg = a.matvec(xd).cpu().numpy(), [o.cpu().numpy() for o in grp.matvec(xd)]
    a.set_prefetch([b])
    grp.set_prefetch([a, b])
    assert np.array_equal(a.matvec(xd).cpu().numpy(), ya)
    assert all(np.array_equal(o.cpu().numpy(), r) for o, r in zip(grp.matvec(xd), yg))
    a.set_prefetch([])
    with pytest.raises(qw.QWeightError):
        a.set_prefetch([b] * 5)


def test_decode_chain_true_dependency():
    """qw_chain: step s reads the y of step s-1 written by other CTAs of the
    same persistent kernel (grid-wide counter); each output equals the
    single-layer launch on the same input and the f64 oracle."""
    torch = _torch()
    la = qw.synth_layer(1024, 1024, seed=80, outlier_ratio=0.005)
    lb = [qw.synth_layer(512, 1024, seed=81 + i, outlier_ratio=0.005) for i in range(2)]
    lc = qw.synth_layer(256, 512, seed=83, group2=4)
    A, B, Cc = qw.DeviceLayer(la), [qw.DeviceLayer(L) for L in lb], qw.DeviceLayer(lc)
    x = torch.from_numpy(qw.synth_activation(1024, 84)).cuda()
    ya = torch.zeros(1024, device="cuda")
    yb = [torch.zeros(512, device="cuda") for _ in range(2)]
    yc = torch.zeros(256, device="cuda")
    ch = qw.DecodeChain([([A], x, [ya], False), (B, ya, yb, True), ([Cc], yb[1], [yc], True)])
    for _ in range(3):  # counters reset per run
        for t in (ya, *yb, yc):
            t.zero_()
        ch.run()
        torch.cuda.synchronize()
        # the chain kernel is the SIMT decode; the per-layer launches may run
        # the tensor-core kernel: equal within the fp16-scale rounding
        ra = A.matvec(x)
        assert rel_l2(ya.cpu().numpy(), ra.cpu().numpy()) <= 2e-3
        for d, o in zip(B, yb):
            assert rel_l2(o.cpu().numpy(), d.matvec(ya).cpu().numpy()) <= 2e-3
        assert rel_l2(yc.cpu().numpy(), Cc.matvec(yb[1]).cpu().numpy()) <= 2e-3
    xa = x.cpu().numpy()
    assert rel_l2(ya.cpu().numpy(), oracle.matvec_f64(la, xa)) <= TOL


@pytest.mark.parametrize("kernel", KERNELS)
def test_decode_chain_llama_shapes_match_group_launches(kernel):
    """The persistent decode chain (SIMT chain kernel, or the warp-MMA chain
    kernel when every layer has the K2m format) equals the group launches."""
    torch = _torch()
    shapes = [(4096, 4096, 3), (4096, 4096, 1), (11008, 4096, 2), (4096, 11008, 1)]
    steps, ref = [], []
    for i, (r, c, n) in enumerate(shapes):
        dls = [qw.DeviceLayer(qw.synth_layer(r, c, seed=90 + 4 * i + j), kernel=kernel) for j in range(n)]
        x = torch.from_numpy(qw.synth_activation(c, 95 + i)).cuda()
        ys = [torch.zeros(r, device="cuda") for _ in range(n)]
        steps.append((dls, x, ys, i > 0))
        ref.append(qw.LayerGroup(dls).matvec(x) if n > 1 else [dls[0].matvec(x)])
    ch = qw.DecodeChain(steps)
    for _ in range(40):  # repeated runs: a slot-ring phase bug once deadlocked ~1 run in 20
        ch.run()
    torch.cuda.synchronize()
    for (dls, x, ys, _), rs in zip(steps, ref):
        for y, r in zip(ys, rs):
            assert rel_l2(y.cpu().numpy(), r.cpu().numpy()) <= 3e-3


def test_decode_chain_rejects_unsupported_geometry():
    torch = _torch()
    d = qw.DeviceLayer(qw.synth_layer(64, 512, seed=1, group2=5))
    x, y = torch.zeros(512, device="cuda"), torch.zeros(64, device="cuda")
    with pytest.raises(qw.QWeightError) as ei:
        qw.DecodeChain([([d], x, [y], False)])
    assert ei.value.status == 5


def test_team_ring_is_race_free():
    """Two teams sharing a slot ring (8192-wide: 25 KB units, a handful of
    slots, 7 units per CTA): every run equals the first and the f64 oracle
    (an odd slot count once let a fast team alias a parity phase)."""
    torch = _torch()
    layer = qw.synth_layer(8192, 8192, seed=7)
    dls = [qw.DeviceLayer(layer)]
    dls.append(dls[0].clone())
    x = torch.from_numpy(qw.synth_activation(8192, 8)).cuda()
    first = dls[0].matvec(x).clone()
    assert rel_l2(first.cpu().numpy(), oracle.matvec_f64(layer, x.cpu().numpy())) <= TOL
    for _ in range(20):
        for d in dls:
            assert torch.equal(d.matvec(x, pdl=True), first)


@pytest.mark.parametrize("kernel", KERNELS)
def test_group_launch_with_unequal_rows_gqa(kernel):
    """GQA-style group: q (512 rows) with k and v (128 rows each) in one launch,
    CTAs split in proportion to the quads; bitwise equal to single launches."""
    torch = _torch()
    layers = [qw.synth_layer(r, 1024, seed=120 + i, outlier_ratio=0.005) for i, r in enumerate((512, 128, 128))]
    dls = [qw.DeviceLayer(L, kernel=kernel) for L in layers]
    grp = qw.LayerGroup(dls)
    x = qw.synth_activation(1024, 121)
    xd = torch.from_numpy(x).cuda()
    outs = grp.matvec(xd)
    for L, d, o in zip(layers, dls, outs):
        assert o.shape[0] == L.cfg.rows
        assert rel_l2(o.cpu().numpy(), oracle.matvec_f64(L, x)) <= TOL
        assert torch.equal(o, d.matvec(xd))


def test_linear_stack_run_end_to_end():
    """LinearStack.run (the e2e API): host inputs -> one graph with the copies
    overlapped -> host outputs; equals the per-layer launches, twice in a row."""
    from paper_2311_16442_b200.stack import LinearStack
    torch = _torch()
    shapes = [(512, 1024), (512, 1024), (256, 512), (1024, 256)]
    layers = [qw.synth_layer(r, c, seed=140 + i) for i, (r, c) in enumerate(shapes)]
    dls = [qw.DeviceLayer(L) for L in layers]
    st = LinearStack(dls, groups=[[0, 1], [2], [3]])
    for trial in range(2):
        xs = [qw.synth_activation(c, 150 + 10 * trial + i) for i, (_, c) in enumerate(shapes)]
        xs[1] = xs[0]  # the fused group reads its first layer's input
        out = st.run(np.concatenate(xs)).copy()
        off = 0
        for d, L, x in zip(dls, layers, xs):
            y = out[off:off + L.cfg.rows]
            off += L.cfg.rows
            assert np.array_equal(y, d.matvec(torch.from_numpy(x).cuda()).cpu().numpy())


def test_auto_kernel_policy():
    """kernel="auto": K2 (SIMT) where it measured faster, K2m (warp MMA) for
    outliers that overflow K2's CSR stage and for layers wider than 16384
    (13B down_proj: K2m at 1 % outliers, K2 at 0.1 %)."""
    dense = qw.synth_layer(5120, 13824, seed=3, outlier_ratio=0.01)  # Llama-2-13B down_proj, 1 %
    sparse = qw.synth_layer(5120, 13824, seed=3, outlier_ratio=0.001)  # the same shape at 0.1 %: K2 fits
    wide = qw.synth_layer(64, 28672, seed=4)
    plain = qw.synth_layer(256, 4096, seed=5)
    assert qw.DeviceLayer(dense).uses_tensor_core
    assert not qw.DeviceLayer(sparse).uses_tensor_core
    assert qw.DeviceLayer(wide).uses_tensor_core
    assert not qw.DeviceLayer(plain).uses_tensor_core
    assert not qw.DeviceLayer(dense, kernel="simt").uses_tensor_core
    assert qw.DeviceLayer(plain, kernel="mma").uses_tensor_core
    x = qw.synth_activation(13824, 6)
    import torch
    y = qw.DeviceLayer(dense).matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel_l2(y, oracle.matvec_f64(dense, x)) <= TOL


@pytest.mark.parametrize("rows,cols,ratio", [(256, 512, 0.01), (512, 4096, 0.005)])
def test_k4_a_tile_is_the_rounded_reference_weight(rows, cols, ratio):
    """every fp16 element of a K4 A tile is RN_fp16 of the
    reference's fp32 weight (reconstruct_dense) times 2^-P.  With a one-hot
    activation at permuted slot k, column n of the batched GEMM is exactly
    A[:, k] * 2^P (one exact product, power-of-two column scales) plus the
    slot's CSR outliers (exact), so y must equal f16(w[:, k] 2^-P) 2^P + csr
    bit for bit."""
    import ctypes as C
    torch = _torch()
    layer = qw.synth_layer(rows, cols, seed=rows + 7, outlier_ratio=ratio)
    dl = qw.DeviceLayer(layer)
    assert dl.batched_path(8) == "gemm", "expected the tcgen05 path"
    P = C.c_int()
    assert qw.lib().qw_debug_gemm_shift(dl._h, C.byref(P)) == 0
    w = oracle.reconstruct_dense(layer)  # rows x padded_cols, permuted order
    perm = layer.plan_perm.astype(np.int64)
    real = np.nonzero(perm != qw.PAD)[0]
    rng = np.random.default_rng(rows)
    slots = np.concatenate([real[:3], rng.choice(real, 5, replace=False)])  # 2-bit and 4-bit slots
    xs = np.zeros((len(slots), cols), np.float32)
    for n, k in enumerate(slots):
        xs[n, perm[k]] = 1.0
    Y = dl.matvec(torch.from_numpy(xs).cuda()).cpu().numpy()
    rp, ci = layer.row_ptr.astype(np.int64), layer.col_ind.astype(np.int64)
    vals = layer.values.view(np.float16).astype(np.float32)
    scale = np.float32(2.0) ** np.float32(P.value)
    for n, k in enumerate(slots):
        a = (w[:, k] / scale).astype(np.float16).astype(np.float32) * scale  # RN_fp16(w 2^-P) 2^P
        csr = np.zeros(rows, np.float32)
        for r in range(rows):
            hit = np.nonzero(ci[rp[r]:rp[r + 1]] == k)[0]
            if hit.size:
                csr[r] = vals[rp[r] + hit[0]]
        expect = a + csr
        assert np.array_equal(Y[n].view(np.uint32), expect.view(np.uint32)), (n, int(k))
