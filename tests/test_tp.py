"""Tensor-parallel split tested on CPU with gloo, world size 2
and 4: the layer is quantized once, sharded column- or row-parallel, each rank
runs the C oracle on its shard, and the NCCL-equivalent collective (all-gather
/ all-reduce over gloo) must reproduce the unsharded result: bitwise for the
column split (rows are independent), to f64 rounding for the row split."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2311_16442_b200 as qw
from paper_2311_16442_b200.tp import TPLinear, split_rows, split_tiles


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
        tp = TPLinear(layer, rank, world, mode, local="oracle")
        y = tp.forward_oracle(x)
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
