"""Tensor-parallel split tested with gloo, world size 2 and 4.

CPU: the layer is quantized once, sharded column- or row-parallel
(paper_2311_16442_b200.tp.shard_layer), each rank runs the C oracle on its
shard, and the collective (all-gather / all-reduce over gloo) must reproduce
the unsharded result: bitwise for the column split (rows are independent), to
f64 rounding for the row split.

GPU (-m gpu): the same ranks (processes sharing cuda:0) run the product
TPLinear.forward -- the repository's kernel on each shard, the gather /
pad / concat and the collective -- at batch 1 and batch 3 and with uneven
splits; compared with the unsharded f64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2311_16442_b200 as qw
from paper_2311_16442_b200.tp import shard_layer, split_rows, split_tiles


def tp_forward_oracle(layer, rank, world, mode, x):
    """The split + collectives with the C oracle as the local matvec."""
    import torch
    shard, ranges, idx = shard_layer(layer, rank, world, mode)
    if mode == "col":
        r0, r1 = ranges[rank]
        local = np.zeros(max(e - s for s, e in ranges), np.float32)
        local[: r1 - r0] = oracle.matvec_oracle(shard, x)
        parts = [torch.zeros_like(torch.from_numpy(local)) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(local))
        return np.concatenate([parts[r].numpy()[: e - s] for r, (s, e) in enumerate(ranges)])
    xs = np.where(idx >= 0, x[np.maximum(idx, 0)], 0.0).astype(np.float32)
    part = torch.from_numpy(oracle.matvec_f64(shard, xs).astype(np.float64))
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    return part.numpy()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, rows, cols, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=0.01)
        x = qw.synth_activation(cols, 77)
        y = tp_forward_oracle(layer, rank, world, mode, x)
        if rank == 0:
            q.put(y)
    finally:
        dist.destroy_process_group()


def _run(world, rows, cols, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, rows, cols, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return y


@pytest.mark.parametrize("world", [2, 4])
def test_column_parallel_all_gather_is_bitwise(world):
    rows, cols = 256, 512
    y = _run(world, rows, cols, "col")
    layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=0.01)
    ref = oracle.matvec_oracle(layer, qw.synth_activation(cols, 77))
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("world", [2, 4])
def test_row_parallel_all_reduce_matches_f64(world):
    rows, cols = 96, 1024
    y = _run(world, rows, cols, "row")
    layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=0.01)
    ref = oracle.matvec_f64(layer, qw.synth_activation(cols, 77))
    assert np.max(np.abs(y - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_split_helpers_cover_the_layer():
    assert split_rows(28672, 16, 8)[-1][1] == 28672
    assert all((e - s) % 16 == 0 for s, e in split_rows(28672, 16, 8))
    r = split_tiles(448, 8)
    assert r[0][0] == 0 and r[-1][1] == 448 and all(e - s == 56 for s, e in r)


# ---------------------------------------------------------------- GPU ranks
def _gpu_worker(rank, world, port, rows, cols, mode, batch, group2, q):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_16442_b200.tp import TPLinear
        layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=0.01, group2=group2)
        xs = np.stack([qw.synth_activation(cols, 77 + b) for b in range(batch)])
        tp = TPLinear(layer, rank, world, mode, device="cuda:0")
        y = tp.forward(torch.from_numpy(xs).cuda()).cpu().numpy()
        if rank == 0:
            q.put(y)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["col", "row"])
@pytest.mark.parametrize("world,rows,cols,batch,group2", [
    (2, 512, 1024, 1, 16),
    (2, 512, 1024, 3, 16),     # batched: the tcgen05 path per shard
    (4, 11008 // 4, 4096, 2, 128),  # column split uneven: 22 row blocks over 4 ranks (ADVICE high)
    (4, 384, 2048, 1, 16),
])
def test_tp_forward_on_gpu_ranks(world, rows, cols, batch, group2, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, rows, cols, mode, batch, group2, q))
             for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    layer = qw.synth_layer(rows, cols, seed=rows + cols, outlier_ratio=0.01, group2=group2)
    for b in range(batch):
        ref = oracle.matvec_f64(layer, qw.synth_activation(cols, 77 + b))
        err = float(np.linalg.norm(y[b] - ref) / np.linalg.norm(ref))
        assert err <= 1e-2, (b, err)


# ------------------------------------------- the exchange fused with the GEMV
def _peer_ranks_in_one_process(layer, world, mode, x):
    """The fused GEMV + peer-memory exchange with `world` ranks as streams of
    ONE process on cuda:0 (same-device ranks in separate processes would need
    MPS for their kernels to run concurrently; between GPUs the peer pointers
    are NVLink P2P / IPC mappings and the kernels are the same).  Returns
    every rank's y."""
    import ctypes as C

    import torch

    from paper_2311_16442_b200._native import check, lib
    from paper_2311_16442_b200.tp import shard_layer
    dls, xs, bufs, flags, ranges = [], [], [], [], None
    for r in range(world):
        shard, ranges_r, idx = shard_layer(layer, r, world, mode)
        ranges = ranges_r or ranges
        dls.append(qw.DeviceLayer(shard, 0, kernel="simt"))
        if mode == "col":
            xs.append(torch.from_numpy(x).cuda())
        else:
            xp = np.concatenate([x, [0.0]]).astype(np.float32)
            xs.append(torch.from_numpy(xp[np.where(idx >= 0, idx, len(x))]).cuda())
        n = layer.cfg.rows if mode == "col" else world * layer.cfg.rows
        bufs.append(torch.zeros(n, dtype=torch.float32, device="cuda"))
        flags.append(torch.zeros(1, dtype=torch.int32, device="cuda"))
    expected = sum(int(lib().qw_push_arrivals(d._h)) for d in dls)
    streams = [torch.cuda.Stream() for _ in range(world)]
    ys = [torch.zeros(layer.cfg.rows, dtype=torch.float32, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    y_loc = [torch.zeros(d.rows, dtype=torch.float32, device="cuda") for d in dls]
    # every push is enqueued before any wait: streams of one process may share
    # a hardware queue, and a spinning wait must not sit ahead of a push
    for r in range(world):
        off = ranges[r][0] if mode == "col" else r * layer.cfg.rows
        peer_y = (C.c_void_p * world)(*[b.data_ptr() + 4 * off for b in bufs])
        peer_f = (C.c_void_p * world)(*[f.data_ptr() for f in flags])
        check(lib().qw_matvec_push(dls[r]._h, C.c_void_p(xs[r].data_ptr()), C.c_void_p(y_loc[r].data_ptr()),
                                   peer_y, peer_f, world, C.c_void_p(streams[r].cuda_stream), 0))
    for r in range(world):
        st = C.c_void_p(streams[r].cuda_stream)
        check(lib().qw_peer_wait(C.c_void_p(flags[r].data_ptr()), expected, st))
        if mode == "row":
            check(lib().qw_peer_reduce(C.c_void_p(bufs[r].data_ptr()), world, layer.cfg.rows,
                                       C.c_void_p(ys[r].data_ptr()), st))
    torch.cuda.synchronize()
    assert all(int(f.item()) == 0 for f in flags)  # every wait took its arrivals off
    for r in range(world):  # the PEER kernel's own y equals the plain kernel's, bit for bit
        plain = dls[r].matvec(xs[r]).cpu().numpy()
        assert np.array_equal(y_loc[r].cpu().numpy().view(np.uint32), plain.view(np.uint32))
    return [(b if mode == "col" else y).cpu().numpy() for b, y in zip(bufs, ys)]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["col", "row"])
@pytest.mark.parametrize("world,rows,cols", [(2, 512, 1024), (3, 11008 // 8, 4096), (4, 384, 2048)])
def test_tp_peer_exchange_fused_with_the_gemv(world, rows, cols, mode):
    """qw_matvec_push (the GEMV whose epilogue stores into every rank's
    buffer and counts its CTAs' arrivals there) + qw_peer_wait (+ the
    rank-order qw_peer_reduce for the row split): every rank ends with the
    full y, equal across ranks and within 1e-2 of the unsharded oracle, for
    two calls in a row (the counters need no reset)."""
    layer = qw.synth_layer(rows, cols, seed=rows + cols + 5, outlier_ratio=0.01)
    for k in range(2):
        x = qw.synth_activation(cols, 80 + k)
        ys = _peer_ranks_in_one_process(layer, world, mode, x)
        ref = oracle.matvec_f64(layer, x)
        for r in range(world):
            err = float(np.linalg.norm(ys[r] - ref) / np.linalg.norm(ref))
            assert err <= 1e-2, (r, k, err)
            assert np.array_equal(ys[r], ys[0])


def _peer_fuzz_cases(n=8, seed=31):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        world = int(rng.integers(2, 7))
        out.append((world, int(rng.integers(world * 16, 2500)), 48 * int(rng.integers(world, 90)),
                    int(rng.choice([4, 16, 32])), str(rng.choice(["col", "row"]))))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world,rows,cols,g2,mode", _peer_fuzz_cases())
def test_tp_peer_exchange_random_geometries(world, rows, cols, g2, mode):
    """The fused peer exchange on seeded random shapes, world sizes and
    2-order group sizes (ranks as streams of one process)."""
    layer = qw.synth_layer(rows, cols, seed=rows * 7 + cols, group2=g2, outlier_ratio=0.005)
    if mode == "row" and (layer.cfg.tail2_blocks or layer.cfg.tail4_blocks):
        pytest.skip("row split needs paired tiles")
    x = qw.synth_activation(cols, rows)
    ys = _peer_ranks_in_one_process(layer, world, mode, x)
    ref = oracle.matvec_f64(layer, x)
    for r in range(world):
        assert float(np.linalg.norm(ys[r] - ref) / np.linalg.norm(ref)) <= 1e-2, r
        assert np.array_equal(ys[r], ys[0])


def _ipc_worker(rank, port, q):
    """Rank 1 maps rank 0's buffer through its CUDA IPC handle and writes into
    it (qw_peer_reduce with one slot); rank 0 reads the values back."""
    import ctypes as C

    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2311_16442_b200._native import check, lib
        buf = torch.zeros(1000, dtype=torch.float32, device="cuda:0")
        torch.cuda.synchronize()
        h = C.create_string_buffer(64)
        check(lib().qw_ipc_handle(C.c_void_p(buf.data_ptr()), h))
        handles = [None, None]
        dist.all_gather_object(handles, h.raw)
        if rank == 1:
            src = torch.arange(1000, dtype=torch.float32, device="cuda:0") * 0.5
            p = C.c_void_p()
            check(lib().qw_ipc_open(handles[0], C.byref(p)))
            check(lib().qw_peer_reduce(C.c_void_p(src.data_ptr()), 1, 1000, p, None))
            torch.cuda.synchronize()
            check(lib().qw_ipc_close(p))
        dist.barrier()
        if rank == 0:
            q.put(buf.cpu().numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ipc_handles_map_a_peer_buffer():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, np.arange(1000, dtype=np.float32) * 0.5)
