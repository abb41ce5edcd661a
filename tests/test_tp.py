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
