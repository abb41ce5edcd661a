"""Tensor-parallel quantized linear over NCCL (BASELINE config 5).

The layer is quantized ONCE as a whole (the outlier top-K, the channel plan
and the 2-order column groups are global: outliers.cpp:81-97, plan.cpp:32-73),
then the packed layer is sharded:

* column-parallel ("col", Megatron q/k/v/gate/up): rank r owns output rows
  [r OC/N, (r+1) OC/N) in whole 2-order row blocks (qw_host_shard_rows); every
  rank reads the full x, computes its rows, and an all-gather assembles y.
* row-parallel ("row", Megatron o/down): rank r owns a contiguous range of
  paired tiles (qw_host_shard_tiles: the tiles' 2-bit triples, 4-bit blocks,
  2-order columns and CSR entries, rebased); its input is the slice of the
  permuted activation those tiles read, and an all-reduce (sum) of the
  partial y gives y.

One process per GPU (torch.distributed); the local GEMV is always this
repository's kernel on the rank's GPU (K2 / K2m at batch 1, K4 at batch
2..16).  The collective runs on the device tensors with NCCL; with a gloo
group (the CPU test harness, several ranks sharing one GPU) the same code
stages the collective's buffers through host memory -- the sharding, gather
and reduction logic is identical.
"""
from __future__ import annotations

import numpy as np

from .layer import PAD, PackedLayer, shard_rows, shard_tiles


def split_rows(rows: int, group2: int, world: int) -> list[tuple[int, int]]:
    """Row ranges per rank, in whole 2-order blocks (the last may be short)."""
    blocks = (rows + group2 - 1) // group2
    out = []
    for r in range(world):
        b0, b1 = blocks * r // world, blocks * (r + 1) // world
        out.append((min(b0 * group2, rows), min(b1 * group2, rows)))
    return out


def split_tiles(tiles: int, world: int) -> list[tuple[int, int]]:
    return [(tiles * r // world, tiles * (r + 1) // world) for r in range(world)]


def shard_layer(layer: PackedLayer, rank: int, world: int, mode: str):
    """The rank's shard of a globally quantized layer.  col: (shard, row
    ranges of every rank, None); row: (shard, None, idx) where idx[i] is the
    original channel shard channel i reads (-1 for a pad: reads 0)."""
    if mode not in ("col", "row"):
        raise ValueError("mode must be 'col' or 'row'")
    if mode == "col":
        ranges = split_rows(layer.cfg.rows, layer.cfg.group2, world)
        r0, r1 = ranges[rank]
        return shard_rows(layer, r0, r1), ranges, None
    if layer.cfg.tail2_blocks or layer.cfg.tail4_blocks:
        raise ValueError("row-parallel split needs paired tiles (T2 == T4)")
    t0, t1 = split_tiles(layer.cfg.triples, world)[rank]
    shard, slots = shard_tiles(layer, t0, t1)
    perm = layer.plan_perm.astype(np.int64)[slots]
    return shard, None, np.where(perm == PAD, -1, perm)


class TPLinear:
    """One rank's shard of a quantized linear + the collective that completes it."""

    def __init__(self, layer: PackedLayer, rank: int, world: int, mode: str, device=None,
                 kernel: str = "auto"):
        import torch

        from .engine import DeviceLayer
        self.mode, self.rank, self.world = mode, rank, world
        self.rows, self.cols = layer.cfg.rows, layer.cfg.cols
        self.shard, self.ranges, self.idx = shard_layer(layer, rank, world, mode)
        self.torch = torch
        dev = torch.device(device if device is not None else "cuda")
        index = dev.index if dev.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", index)
        self.dl = DeviceLayer(self.shard, index, kernel=kernel)
        if self.idx is not None:
            # one gather from x padded with a zero column: pads read it
            self.gidx = torch.from_numpy(np.where(self.idx >= 0, self.idx, self.cols)).to(self.device)
        self.max_rows = max(r1 - r0 for r0, r1 in self.ranges) if mode == "col" else self.rows

    def _collective(self, fn, *tensors, group=None):
        """Run a collective on device tensors (NCCL) or, for a gloo group,
        through host copies (the multi-rank CPU harness)."""
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            fn(*tensors)
            return tensors
        host = [t.cpu() if isinstance(t, self.torch.Tensor) else [u.cpu() for u in t] for t in tensors]
        fn(*host)
        return host

    def forward(self, x, group=None):
        """x: full activation(s) in original channel order, cuda fp32
        [cols] or [batch, cols], identical on every rank.  Returns the full y
        on the rank's device."""
        torch = self.torch
        import torch.distributed as dist
        squeeze = x.dim() == 1
        xb = (x.reshape(1, -1) if squeeze else x).to(self.device)
        b = xb.shape[0]
        if self.mode == "col":
            r0, r1 = self.ranges[self.rank]
            y_loc = torch.zeros(b, self.max_rows, dtype=torch.float32, device=self.device)
            y_loc[:, : r1 - r0] = self.dl.matvec(xb)  # contiguous [b, r1 - r0] first
            gathered = torch.empty(self.world * b, self.max_rows, dtype=torch.float32, device=self.device)
            out = self._collective(lambda o, i: dist.all_gather_into_tensor(o, i, group=group),
                                   gathered, y_loc, group=group)[0]
            out = out.to(self.device).reshape(self.world, b, self.max_rows)
            y = torch.cat([out[r, :, : e - s] for r, (s, e) in enumerate(self.ranges)], dim=1)
        else:
            xp = torch.cat([xb, torch.zeros(b, 1, dtype=xb.dtype, device=self.device)], dim=1)
            y = self.dl.matvec(xp.index_select(1, self.gidx))
            y = self._collective(lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group),
                                 y, group=group)[0].to(self.device)
        return y.reshape(-1) if squeeze else y
