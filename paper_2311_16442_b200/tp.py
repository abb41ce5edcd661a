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
    """One rank's shard of a quantized linear + the exchange that completes it.

    exchange="collective": NCCL all-gather / all-reduce (or gloo through host
    memory in the CPU harness).  exchange="peer" (batch 1; larger batches use
    the collective): the exchange is fused with the GEMV -- the kernel's
    epilogue stores this rank's rows straight into every rank's buffer
    (column split: its rows of every rank's full y; row split: its partial
    into its slot of every rank's staging buffer) over CUDA IPC mappings
    (NVLink P2P between GPUs) and adds its CTAs' arrivals to every rank's
    counter; one stream-ordered wait (and, for the row split, the rank-order
    sum of the slots) completes it.  The buffers are exchanged once, at
    construction, through the process group (collective call: every rank
    constructs its TPLinear together).  The returned y is this layer's
    buffer, rewritten by its next call.  One rank per GPU (the wait kernel
    spins until the other ranks' kernels have pushed; ranks sharing a GPU
    from separate processes would need MPS to run concurrently -- the tests
    run such ranks as streams of one process, tests/test_tp.py)."""

    def __init__(self, layer: PackedLayer, rank: int, world: int, mode: str, device=None,
                 kernel: str = "auto", exchange: str = "collective", group=None):
        import torch

        from .engine import DeviceLayer
        if exchange not in ("collective", "peer"):
            raise ValueError("exchange must be 'collective' or 'peer'")
        self.mode, self.rank, self.world, self.exchange = mode, rank, world, exchange
        self.rows, self.cols = layer.cfg.rows, layer.cfg.cols
        self.shard, self.ranges, self.idx = shard_layer(layer, rank, world, mode)
        self.torch = torch
        dev = torch.device(device if device is not None else "cuda")
        index = dev.index if dev.index is not None else torch.cuda.current_device()
        self.device = torch.device("cuda", index)
        # the fused exchange runs on the SIMT kernel
        self.dl = DeviceLayer(self.shard, index, kernel="simt" if exchange == "peer" else kernel)
        if self.idx is not None:
            # one gather from x padded with a zero column: pads read it
            self.gidx = torch.from_numpy(np.where(self.idx >= 0, self.idx, self.cols)).to(self.device)
        self.max_rows = max(r1 - r0 for r0, r1 in self.ranges) if mode == "col" else self.rows
        if exchange == "peer":
            self._bind_peers(group)

    def _bind_peers(self, group):
        """Allocate this rank's exchange buffers, swap CUDA IPC handles with
        the other ranks and point the kernel's peer stores at their buffers."""
        import ctypes as C

        import torch.distributed as dist

        from ._native import check, lib
        torch = self.torch
        n = self.rows if self.mode == "col" else self.world * self.rows
        self.xbuf = torch.zeros(n, dtype=torch.float32, device=self.device)      # full y / staging slots
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)        # arrival counter
        self.y_out = self.xbuf if self.mode == "col" else torch.zeros(self.rows, dtype=torch.float32,
                                                                       device=self.device)
        self.y_loc = torch.zeros(self.dl.rows, dtype=torch.float32, device=self.device)
        torch.cuda.synchronize(self.device)

        def handle(t):
            h = C.create_string_buffer(64)
            check(lib().qw_ipc_handle(C.c_void_p(t.data_ptr()), h))
            return h.raw

        mine = (handle(self.xbuf), handle(self.flag), int(lib().qw_push_arrivals(self.dl._h)))
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.expected = sum(e[2] for e in everyone)
        self._opened = []
        ys, flags = [], []
        for r, (hb, hf, _) in enumerate(everyone):
            if r == self.rank:
                base, fl = self.xbuf.data_ptr(), self.flag.data_ptr()
            else:
                pb, pf = C.c_void_p(), C.c_void_p()
                check(lib().qw_ipc_open(hb, C.byref(pb)))
                check(lib().qw_ipc_open(hf, C.byref(pf)))
                self._opened += [pb.value, pf.value]
                base, fl = pb.value, pf.value
            off = self.ranges[self.rank][0] if self.mode == "col" else self.rank * self.rows
            ys.append(base + 4 * off)
            flags.append(fl)
        self._peer_y = (C.c_void_p * self.world)(*ys)
        self._peer_flag = (C.c_void_p * self.world)(*flags)
        dist.barrier(group=group)

    def close(self):
        """Unmap the peers' buffers (peer exchange)."""
        import ctypes as C

        from ._native import lib
        for p in getattr(self, "_opened", []):
            lib().qw_ipc_close(C.c_void_p(p))
        self._opened = []

    def _forward_peer(self, xb):
        """Batch 1 over peer memory: one fused GEMV + exchange launch, the wait
        for every rank's arrivals, and (row split) the rank-order sum."""
        import ctypes as C

        from ._native import check, lib
        from .engine import _stream_handle
        torch = self.torch
        stream = C.c_void_p(_stream_handle(None))
        if self.mode == "col":
            x = xb.reshape(-1).contiguous()
        else:
            xp = torch.cat([xb, torch.zeros(1, 1, dtype=xb.dtype, device=self.device)], dim=1)
            x = xp.index_select(1, self.gidx).reshape(-1).contiguous()
        check(lib().qw_matvec_push(self.dl._h, C.c_void_p(x.data_ptr()), C.c_void_p(self.y_loc.data_ptr()),
                                   self._peer_y, self._peer_flag, self.world, stream, 0))
        check(lib().qw_peer_wait(C.c_void_p(self.flag.data_ptr()), self.expected, stream))
        if self.mode == "row":
            check(lib().qw_peer_reduce(C.c_void_p(self.xbuf.data_ptr()), self.world, self.rows,
                                       C.c_void_p(self.y_out.data_ptr()), stream))
        return self.y_out.reshape(1, -1)

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
        if self.exchange == "peer" and b == 1:
            y = self._forward_peer(xb)
            return y.reshape(-1) if squeeze else y
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
