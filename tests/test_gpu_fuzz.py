"""Seeded random geometries through every device path against the f64
oracle: 64 small (rows 1..700, any residue mod 4; cols a multiple of 16 up
to 2560), 16 large (rows up to 6000, cols up to 14336) and 8 very wide
(cols 16384..30720: x gathered from global memory) layers,
alpha 0 / 0.25 / 0.5 / 1 (pure 2-bit to pure 4-bit), group2 1..128 (row
blocks that do and do not align with quads), outlier ratio 0..2 %.  Per case and
batch-1 kernel (the default choice, K2 and K2m forced): batch 1 (rel-L2 and
normwise max within the north-star 1e-2) and a column launch of a random
batch (every column bit-identical to its batch-1 call); with the default
upload the tcgen05 GEMM K4 at that batch (within 1e-2, deterministic run to
run).  A layer K2's shared-memory plan cannot take is refused cleanly when
K2 is forced and served by K2m by default.  Also 24 random layer groups
(GQA-style differing rows, batch 1..8, each output bit-identical to the
layer's own launch) and 16 random tensor-parallel shardings (column / row
split over 2..8 ranks, exchange completed on the host), 24 random shapes
through the GPU producer (QWL1 bytes identical to the CPU producer's) and 16
random tcgen05 geometries for the A-tile exactness, and 12 random
persistent decode chains (dependent steps, K2 and K2m chain kernels) and 8
random back-to-back PDL chains (bit-identical to synchronised calls) and 8
random layers loaded straight from QWL1 containers."""
import os

import numpy as np
import pytest

import oracle
import paper_2311_16442_b200 as qw

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _cases(n=64, seed=2311, max_rows=700, max_cols16=160, first=0):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(first, first + n):
        rows = int(rng.integers(1, max_rows + 1))
        cols = 16 * int(rng.integers(1, max_cols16 + 1))
        alpha = float(rng.choice([0.0, 0.25, 0.25, 0.5, 1.0]))
        group2 = int(rng.choice([1, 3, 4, 5, 8, 16, 16, 32, 128]))
        ratio = float(rng.choice([0.0, 0.001, 0.005, 0.01, 0.02]))
        batch = int(rng.integers(2, 17))
        out.append((i, rows, cols, alpha, group2, ratio, batch))
    return out


def _check(y, ref, what):
    ref = np.asarray(ref, np.float64)
    assert np.all(np.isfinite(y)), what
    den = np.linalg.norm(ref)
    err = float(np.linalg.norm(np.asarray(y, np.float64) - ref) / (den if den else 1.0))
    assert err <= TOL, (what, err)
    scale = np.max(np.abs(ref)) if ref.size else 0.0
    assert np.max(np.abs(y - ref)) <= TOL * max(scale, 1e-30) + 1e-30, what


# small layers (every residue, tails, tiny grids) and large ones (wide rows,
# many CTAs, stream-K / split-K GEMM schedules)
# QW_FUZZ_N / QW_FUZZ_SEED: a longer or different draw of the small layers (stress runs)
_N, _SEED = int(os.environ.get("QW_FUZZ_N", "64")), int(os.environ.get("QW_FUZZ_SEED", "2311"))
CASES = (_cases(n=_N, seed=_SEED) + _cases(n=16, seed=1644, max_rows=6000, max_cols16=896, first=_N) +
         # wider than the 16384 channels K2 stages in shared memory (x gathered from global memory)
         [c for c in _cases(n=40, seed=4242, max_rows=300, max_cols16=1920, first=_N + 16) if c[2] > 16384][:8])


@pytest.mark.parametrize("case", CASES, ids=lambda c: "r{1}c{2}a{3}g{4}o{5}b{6}".format(*c))
def test_random_geometry_all_paths(case):
    import torch
    i, rows, cols, alpha, group2, ratio, batch = case
    layer = qw.synth_layer(rows, cols, seed=1000 + i, alpha=alpha, group2=group2, outlier_ratio=ratio)
    xs = np.stack([qw.synth_activation(cols, 2000 + 17 * i + b) for b in range(batch)])
    refs = [oracle.matvec_f64(layer, xs[b]) for b in range(batch)]
    X = torch.from_numpy(xs).cuda()
    for kernel in ("auto", "simt", "mma"):
        try:
            dl = qw.DeviceLayer(layer, kernel=kernel)
        except qw.QWeightError as e:
            # the SIMT kernel's shared-memory plan may not fit a wide layer:
            # a clean refusal, and the default upload serves it with K2m
            assert kernel == "simt" and e.status == 5, (kernel, str(e))
            continue
        y1 = dl.matvec(X[0].contiguous()).cpu().numpy()
        _check(y1, refs[0], f"{kernel} batch 1")
        yc = dl.matvec(X, batched="columns").cpu().numpy()
        for b in range(batch):
            yb = dl.matvec(X[b].contiguous()).cpu().numpy()
            assert np.array_equal(yc[b].view(np.uint32), yb.view(np.uint32)), (kernel, "column launch", b)
            _check(yc[b], refs[b], f"{kernel} column {b}")
        if kernel == "auto" and dl.batched_path(batch, "gemm") == "gemm":
            yg = dl.matvec(X, batched="gemm").cpu().numpy()
            for b in range(batch):
                _check(yg[b], refs[b], f"K4 column {b}")
            assert np.array_equal(yg, dl.matvec(X, batched="gemm").cpu().numpy()), "K4 not deterministic"
        dl.close()


def _group_cases(n=24, seed=77):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        cols = 16 * int(rng.integers(1, 257))
        nl = int(rng.integers(2, 4))
        rows = [int(rng.integers(1, 1500)) for _ in range(nl)]
        alpha = float(rng.choice([0.0, 0.25, 0.5, 1.0]))
        group2 = int(rng.choice([3, 4, 16, 16, 32]))
        ratio = float(rng.choice([0.0, 0.002, 0.01]))
        batch = int(rng.integers(1, 9))
        kernel = str(rng.choice(["auto", "simt", "mma"]))
        out.append((i, cols, tuple(rows), alpha, group2, ratio, batch, kernel))
    return out


@pytest.mark.parametrize("case", _group_cases(), ids=lambda c: "c{1}r{2}a{3}g{4}o{5}b{6}{7}".format(*c))
def test_random_layer_group(case):
    """A layer group (GQA-style: the row counts differ) at batch 1 or a batch:
    every output bit-identical to the layer's own launch and within 1e-2 of
    the oracle."""
    import torch
    i, cols, rows, alpha, group2, ratio, batch, kernel = case
    # one channel split for the group: the same calibration vector for every layer
    h = qw.synth_calibration(cols, 900 + i)
    layers = [qw.quantize_layer(qw.synth_gaussian(r, cols, 600 + 10 * i + j), h, alpha, group2, ratio)
              for j, r in enumerate(rows)]
    try:
        dls = [qw.DeviceLayer(L, kernel=kernel) for L in layers]
    except qw.QWeightError as e:
        assert kernel == "simt" and e.status == 5, str(e)
        return
    grp = qw.LayerGroup(dls)
    xs = np.stack([qw.synth_activation(cols, 3000 + 13 * i + b) for b in range(batch)])
    X = torch.from_numpy(xs).cuda()
    x_in = X[0].contiguous() if batch == 1 else X
    outs = [o.cpu().numpy().reshape(batch, -1) for o in grp.matvec(x_in)]
    for L, dl, o in zip(layers, dls, outs):
        own = dl.matvec(x_in).cpu().numpy().reshape(batch, -1) if batch == 1 else None
        for b in range(batch):
            ref = oracle.matvec_f64(L, xs[b])
            _check(o[b], ref, f"group layer rows {L.cfg.rows} column {b}")
            yb = dl.matvec(X[b].contiguous()).cpu().numpy()
            assert np.array_equal(o[b].view(np.uint32), yb.view(np.uint32)), ("group vs own launch", b)
        if own is not None:
            assert np.array_equal(own, o)
    grp.close()


def _tp_cases(n=16, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        world = int(rng.integers(2, 9))
        mode = str(rng.choice(["col", "row"]))
        rows = int(rng.integers(world * 16, 3000))
        cols = 48 * int(rng.integers(world, 80))  # whole triples: paired tiles for the row split
        group2 = int(rng.choice([4, 16, 16, 32]))
        ratio = float(rng.choice([0.0, 0.002, 0.01]))
        out.append((i, world, mode, rows, cols, group2, ratio))
    return out


@pytest.mark.parametrize("case", _tp_cases(), ids=lambda c: "w{1}{2}r{3}c{4}g{5}o{6}".format(*c))
def test_random_tensor_parallel_shards(case):
    """Quantize once, shard (column split: row ranges on 2-order block
    boundaries; row split: whole tile pairs), run every shard's GPU matvec and
    complete the exchange on the host (concatenate / sum in rank order): the
    result is within 1e-2 of the unsharded layer's f64 oracle."""
    import torch

    from paper_2311_16442_b200.tp import shard_layer
    i, world, mode, rows, cols, group2, ratio = case
    layer = qw.synth_layer(rows, cols, seed=700 + i, alpha=0.25, group2=group2, outlier_ratio=ratio)
    if mode == "row" and (layer.cfg.tail2_blocks or layer.cfg.tail4_blocks):
        pytest.skip("row split needs paired tiles")
    x = qw.synth_activation(cols, 800 + i)
    ref = oracle.matvec_f64(layer, x)
    parts = []
    for r in range(world):
        shard, ranges, idx = shard_layer(layer, r, world, mode)
        xs = x if mode == "col" else np.where(idx >= 0, x[np.maximum(idx, 0)], 0.0).astype(np.float32)
        y = qw.DeviceLayer(shard).matvec(torch.from_numpy(np.ascontiguousarray(xs)).cuda()).cpu().numpy()
        parts.append(y)
    if mode == "col":
        got = np.concatenate(parts)
    else:
        got = parts[0].astype(np.float32).copy()
        for p in parts[1:]:
            got += p
    assert got.shape == ref.shape
    _check(got, ref, f"{mode} split over {world}")


def _producer_cases(n=24, seed=5):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        rows = int(rng.integers(1, 1200))
        cols = 16 * int(rng.integers(1, 200))
        alpha = float(rng.choice([0.0, 0.125, 0.25, 0.5, 0.75, 1.0]))
        group2 = int(rng.choice([1, 2, 3, 5, 8, 16, 64, 128]))
        ratio = float(rng.choice([0.0, 0.0005, 0.002, 0.01, 0.05]))
        ties = bool(rng.integers(0, 2))
        out.append((i, rows, cols, alpha, group2, ratio, ties))
    return out


@pytest.mark.parametrize("case", _producer_cases(), ids=lambda c: "r{1}c{2}a{3}g{4}o{5}t{6}".format(*c))
def test_random_device_producer_bit_identical(case, tmp_path):
    """qw_device_quantize vs the CPU producer (itself pinned to the
    reference) on random shapes, as serialized QWL1 bytes; half the cases
    plant equal-magnitude outliers to exercise the top-K tie-break."""
    i, rows, cols, alpha, group2, ratio, ties = case
    w = qw.synth_gaussian(rows, cols, 4000 + i)
    if ties:
        rng = np.random.default_rng(i)
        for _ in range(min(8, rows * cols // 4)):
            w[int(rng.integers(0, rows)), int(rng.integers(0, cols))] = 7.5  # exact ties in |w|
    h = qw.synth_calibration(cols, 4100 + i)
    cpu = qw.quantize_layer(w, h, alpha, group2, ratio)
    gpu = qw.quantize_layer_gpu(w, h, alpha, group2, ratio)
    pc, pg = tmp_path / "cpu.qwl", tmp_path / "gpu.qwl"
    qw.write_packed_layer(cpu, str(pc))
    qw.write_packed_layer(gpu, str(pg))
    assert pg.read_bytes() == pc.read_bytes()


def _a_tile_cases(n=16, seed=11):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        rows = int(rng.integers(1, 2000))
        cols = 128 * int(rng.integers(1, 40))
        group2 = int(rng.choice([4, 8, 16, 16, 32, 128]))
        ratio = float(rng.choice([0.0, 0.002, 0.01]))
        out.append((i, rows, cols, group2, ratio))
    return out


@pytest.mark.parametrize("case", _a_tile_cases(), ids=lambda c: "r{1}c{2}g{3}o{4}".format(*c))
def test_random_k4_a_tile_exactness(case):
    """SURVEY §8(c)(2) on random K4 geometries: with a one-hot activation at
    permuted slot k, column n of the batched GEMM equals
    RN_fp16(w[:, k] 2^-P) 2^P plus the slot's CSR outliers, bit for bit
    (tests/test_gpu_parity.py states the argument)."""
    import ctypes as C

    import torch
    i, rows, cols, group2, ratio = case
    layer = qw.synth_layer(rows, cols, seed=5000 + i, group2=group2, outlier_ratio=ratio)
    dl = qw.DeviceLayer(layer)
    if dl.batched_path(8, "gemm") != "gemm":
        pytest.skip("geometry not on the tcgen05 path (unpaired tiles)")
    P = C.c_int()
    assert qw.lib().qw_debug_gemm_shift(dl._h, C.byref(P)) == 0
    w = oracle.reconstruct_dense(layer)
    perm = layer.plan_perm.astype(np.int64)
    real = np.nonzero(perm != qw.PAD)[0]
    rng = np.random.default_rng(6000 + i)
    slots = rng.choice(real, min(8, real.size), replace=False)
    xs = np.zeros((len(slots), cols), np.float32)
    for n, k in enumerate(slots):
        xs[n, perm[k]] = 1.0
    Y = dl.matvec(torch.from_numpy(xs).cuda(), batched="gemm").cpu().numpy()
    rp, ci = layer.row_ptr.astype(np.int64), layer.col_ind.astype(np.int64)
    vals = layer.values.view(np.float16).astype(np.float32)
    scale = np.float32(2.0) ** np.float32(P.value)
    for n, k in enumerate(slots):
        a = (w[:, k] / scale).astype(np.float16).astype(np.float32) * scale
        csr = np.zeros(rows, np.float32)
        for r in range(rows):
            hit = np.nonzero(ci[rp[r]:rp[r + 1]] == k)[0]
            if hit.size:
                csr[r] = vals[rp[r] + hit[0]]
        assert np.array_equal(Y[n].view(np.uint32), (a + csr).view(np.uint32)), (n, int(k))


def _chain_cases(n=12, seed=21):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        steps = int(rng.integers(2, 6))
        dims = [16 * int(rng.integers(4, 200)) for _ in range(steps + 1)]  # x width of each step, then the last y
        extra = [int(rng.integers(0, 3)) for _ in range(steps)]           # more layers reading the same x
        kernel = str(rng.choice(["simt", "mma"]))
        out.append((i, tuple(dims), tuple(extra), kernel))
    return out


@pytest.mark.parametrize("case", _chain_cases(), ids=lambda c: "d{1}e{2}{3}".format(*c).replace(" ", ""))
def test_random_decode_chain(case):
    """The persistent chain kernel (DecodeChain) over random dependent steps:
    step s reads the output of step s-1's first layer; every output within
    1e-2 of the oracle applied to the chain's own input of that step, and run
    to run deterministic."""
    import torch
    i, dims, extra, kernel = case
    steps, keep = [], []
    x0 = torch.from_numpy(qw.synth_activation(dims[0], 7000 + i)).cuda()
    x = x0
    for s in range(len(dims) - 1):
        cols = dims[s]
        # the SIMT chain kernel takes one geometry per step, the K2m one differing rows (GQA)
        rows = [dims[s + 1]] + [dims[s + 1] if kernel == "simt" else 16 * (1 + (s + j) % 5)
                                for j in range(extra[s])]
        h = qw.synth_calibration(cols, 7100 + 10 * i + s)
        layers = [qw.quantize_layer(qw.synth_gaussian(r, cols, 7200 + 100 * i + 10 * s + j), h, 0.25, 16, 0.005)
                  for j, r in enumerate(rows)]
        dls = [qw.DeviceLayer(L, kernel=kernel) for L in layers]
        ys = [torch.empty(r, device="cuda") for r in rows]
        steps.append((dls, x, ys, s > 0))
        keep.append((layers, x, ys))
        x = ys[0]
    try:
        chain = qw.DecodeChain(steps)
    except qw.QWeightError as e:
        assert e.status == 5, str(e)  # a geometry the chain kernel does not cover: refused cleanly
        pytest.skip(str(e))
    chain.run()
    torch.cuda.synchronize()
    first = [[y.cpu().numpy().copy() for y in ys] for _, _, ys in keep]
    for s, (layers, xin, ys) in enumerate(keep):
        xv = xin.cpu().numpy()
        for L, y in zip(layers, ys):
            _check(y.cpu().numpy(), oracle.matvec_f64(L, xv), f"chain step {s}")
    chain.run()
    torch.cuda.synchronize()
    for s, (_, _, ys) in enumerate(keep):
        for a, y in zip(first[s], ys):
            assert np.array_equal(a, y.cpu().numpy()), ("chain not deterministic", s)
    chain.close()


@pytest.mark.parametrize("seed", range(8))
def test_random_pdl_chains_match_synchronised_calls(seed):
    """Back-to-back dependent launches with programmatic dependent launch
    (each call reads the previous call's y; the next kernel starts under the
    previous one and waits in griddepcontrol.wait) on random shapes, batch 1
    and batched (column launches / K4), K2 and K2m: bit-identical to the same
    calls with a device synchronisation between them."""
    import torch
    rng = np.random.default_rng(8800 + seed)
    kernel = str(rng.choice(["simt", "mma", "auto"]))
    batch = int(rng.choice([1, 1, 3, 8]))
    dims = [16 * int(rng.integers(8, 300)) for _ in range(6)]
    dls = [qw.DeviceLayer(qw.synth_layer(dims[s + 1], dims[s], seed=8900 + 10 * seed + s, outlier_ratio=0.005),
                          kernel=kernel) for s in range(5)]
    x0 = np.stack([qw.synth_activation(dims[0], 9000 + seed + b) for b in range(batch)])
    X0 = torch.from_numpy(x0 if batch > 1 else x0[0]).cuda()
    ref, x = [], X0
    for d in dls:  # synchronised
        x = d.matvec(x)
        torch.cuda.synchronize()
        ref.append(x.cpu().numpy())
    got, x = [], X0
    for d in dls:  # back to back under PDL
        x = d.matvec(x, pdl=True)
        got.append(x)
    torch.cuda.synchronize()
    for s in range(5):
        assert np.array_equal(got[s].cpu().numpy(), ref[s]), (kernel, batch, s)


@pytest.mark.parametrize("seed", range(8))
def test_random_qwl_straight_to_device(seed, tmp_path):
    """A random layer written as a QWL1 container and loaded straight into
    HBM (qw_layer_load / qw_layer_upload_qwl: parse, CRC, validate, repack)
    computes the same y, bit for bit, as the in-memory upload."""
    import torch
    rng = np.random.default_rng(9500 + seed)
    rows, cols = int(rng.integers(1, 3000)), 16 * int(rng.integers(1, 600))
    layer = qw.synth_layer(rows, cols, seed=9600 + seed, alpha=float(rng.choice([0.0, 0.25, 1.0])),
                           group2=int(rng.choice([1, 5, 16, 128])), outlier_ratio=float(rng.choice([0.0, 0.005])))
    path = tmp_path / "layer.qwl"
    qw.write_packed_layer(layer, str(path))
    x = torch.from_numpy(qw.synth_activation(cols, seed)).cuda()
    y = qw.DeviceLayer(layer).matvec(x).cpu().numpy()
    for dl in (qw.DeviceLayer.load(str(path)), qw.DeviceLayer.from_qwl_bytes(path.read_bytes())):
        assert np.array_equal(dl.matvec(x).cpu().numpy().view(np.uint32), y.view(np.uint32))
