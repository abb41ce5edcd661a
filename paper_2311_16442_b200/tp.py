"""Tensor-parallel quantized linear over NCCL (BASELINE config 5).

The layer is quantized ONCE as a whole (the outlier top-K, the channel plan
and the 2-order column groups are global: outliers.cpp:81-97, plan.cpp:32-73),
then the packed layer is sharded:

* column-parallel ("col", Megatron q/k/v/gate/up): rank r owns output rows
  [r OC/N, (r+1) OC/N) in whole 2-order row blocks (qw_host_shard_rows); every
  rank reads the full x, computes its rows, and an NCCL all-gather assembles y.
* row-parallel ("row", Megatron o/down): rank r owns a contiguous range of
  paired tiles (qw_host_shard_tiles: the tiles' 2-bit triples, 4-bit blocks,
  2-order columns and CSR entries, rebased); its input is the slice of the
  permuted activation those tiles read, and an NCCL all-reduce (sum) of the
  partial y gives y.

One process per GPU (torch.distributed, backend "nccl"); the local GEMV is
the fused K2 kernel (batch 1) or K4 (batch 2..16).  The same class runs on
CPU with backend "gloo" and the C oracle as the local matvec (test only:
`local="oracle"`), which is how the sharding + collective logic is tested
without GPUs.
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


class TPLinear:
    """One rank's shard of a quantized linear + the collective that completes it."""

    def __init__(self, layer: PackedLayer, rank: int, world: int, mode: str, device=None,
                 local: str = "gpu"):
        if mode not in ("col", "row"):
            raise ValueError("mode must be 'col' or 'row'")
        self.mode, self.rank, self.world, self.local = mode, rank, world, local
        self.rows, self.cols = layer.cfg.rows, layer.cfg.cols
        if mode == "col":
            self.ranges = split_rows(self.rows, layer.cfg.group2, world)
            r0, r1 = self.ranges[rank]
            self.shard = shard_rows(layer, r0, r1)
            self.idx = None
        else:
            if layer.cfg.tail2_blocks or layer.cfg.tail4_blocks:
                raise ValueError("row-parallel split needs paired tiles (T2 == T4)")
            t0, t1 = split_tiles(layer.cfg.triples, world)[rank]
            self.shard, slots = shard_tiles(layer, t0, t1)
            perm = layer.plan_perm.astype(np.int64)[slots]
            # shard channel i reads original channel perm[i]; pads read 0
            self.idx = np.where(perm == PAD, -1, perm)
        self.dev = None
        if local == "gpu":
            import torch

            from .engine import DeviceLayer
            self.torch = torch
            self.device = torch.device(device if device is not None else "cuda")
            self.dl = DeviceLayer(self.shard, self.device.index or 0)
            if self.idx is not None:
                real = self.idx >= 0
                self.gidx = torch.from_numpy(np.where(real, self.idx, 0)).to(self.device)
                self.gmask = torch.from_numpy(real.astype(np.float32)).to(self.device)
            self.max_rows = max(r1 - r0 for r0, r1 in self.ranges) if mode == "col" else self.rows

    # ------------------------------------------------------------------ GPU
    def forward(self, x, group=None):
        """x: full activation(s) in original channel order, cuda fp32
        [cols] or [batch, cols], identical on every rank.  Returns the full y."""
        torch = self.torch
        import torch.distributed as dist
        squeeze = x.dim() == 1
        xb = x.reshape(1, -1) if squeeze else x
        b = xb.shape[0]
        if self.mode == "col":
            r0, r1 = self.ranges[self.rank]
            y_loc = torch.zeros(b, self.max_rows, dtype=torch.float32, device=self.device)
            self.dl.matvec(xb, out=y_loc[:, : r1 - r0])
            gathered = torch.empty(self.world, b, self.max_rows, dtype=torch.float32, device=self.device)
            dist.all_gather_into_tensor(gathered, y_loc, group=group)
            y = torch.cat([gathered[r, :, : e - s] for r, (s, e) in enumerate(self.ranges)], dim=1)
        else:
            xs = (xb.index_select(1, self.gidx) * self.gmask).contiguous()
            y = self.dl.matvec(xs)
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        return y.reshape(-1) if squeeze else y

    # ------------------------------------------------------------------ CPU (tests)
    def forward_oracle(self, x: np.ndarray, group=None) -> np.ndarray:
        """Same split + collectives with the C oracle as the local matvec
        (gloo on CPU).  Test infrastructure: imports oracle lazily."""
        import torch
        import torch.distributed as dist

        import oracle
        if self.mode == "col":
            r0, r1 = self.ranges[self.rank]
            local = np.zeros(max(e - s for s, e in self.ranges), np.float32)
            local[: r1 - r0] = oracle.matvec_oracle(self.shard, x)
            parts = [torch.zeros_like(torch.from_numpy(local)) for _ in range(self.world)]
            dist.all_gather(parts, torch.from_numpy(local), group=group)
            return np.concatenate([parts[r].numpy()[: e - s] for r, (s, e) in enumerate(self.ranges)])
        xs = np.where(self.idx >= 0, x[np.maximum(self.idx, 0)], 0.0).astype(np.float32)
        part = torch.from_numpy(oracle.matvec_f64(self.shard, xs).astype(np.float64))
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
        return part.numpy()
