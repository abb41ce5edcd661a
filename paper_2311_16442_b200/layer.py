"""Host-side packed layer and producer, mirroring the reference host API.

`PackedLayer` mirrors qweight::PackedLayer (reference bitpack.hpp:112-124)
with numpy arrays for its streams; sorder/fourbit are kept as
structure-of-arrays (the C-ABI view layout).  The producer functions
(`synth_*`, `quantize_layer`, `read_packed_layer`, ...) call the native host
library, whose results are bit-identical to the reference (pinned by
tests/test_producer.py against the compiled reference).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._native import LayerInfo, LayerView, QWeightError, check, lib

PAD = 0xFFFFFFFF  # kPadChannel (plan.hpp:12)
G1, TILE, TILE2, TILE4 = 16, 64, 48, 16


@dataclass
class LayerConfig:
    """qweight::LayerConfig (bitpack.hpp:59-98)."""
    rows: int
    cols: int
    n4: int
    pad2: int
    outlier_count: int = 0
    group2: int = 16
    alpha: float = 0.0
    outlier_ratio: float = 0.0
    n: int = 2
    n2: int = 4
    group1: int = 16
    tile: int = 64

    @property
    def n2_padded(self): return self.cols - self.n4 + self.pad2
    @property
    def padded_cols(self): return self.n2_padded + self.n4
    @property
    def triples(self): return self.n2_padded // TILE2
    @property
    def blocks4(self): return self.n4 // TILE4
    @property
    def paired(self): return min(self.triples, self.blocks4)
    @property
    def tail2_blocks(self): return self.triples - self.paired
    @property
    def tail4_blocks(self): return self.blocks4 - self.paired
    @property
    def groups_per_row(self): return 3 * self.triples
    @property
    def row_blocks(self): return (self.rows + self.group2 - 1) // self.group2


@dataclass
class PackedLayer:
    cfg: LayerConfig
    plan_bits: np.ndarray
    plan_perm: np.ndarray
    main: np.ndarray
    tail2: np.ndarray
    tail4: np.ndarray
    secondary: np.ndarray
    meta: np.ndarray
    sorder_zero2: np.ndarray
    sorder_scale2: np.ndarray
    fourbit_scale: np.ndarray
    fourbit_zero: np.ndarray
    row_ptr: np.ndarray
    col_ind: np.ndarray
    values: np.ndarray
    _keep: list = field(default_factory=list, repr=False, compare=False)

    # ------------------------------------------------------------ views
    def view(self) -> LayerView:
        """Borrowed C view; valid while this object is alive."""
        c = self.cfg
        v = LayerView()
        for k in ("n", "n2", "group1", "group2", "tile", "rows", "cols", "n4", "pad2",
                  "outlier_count", "alpha", "outlier_ratio"):
            setattr(v, k, getattr(c, k))
        arrays = {
            "plan_bits": (self.plan_bits, np.uint8), "plan_perm": (self.plan_perm, np.uint32),
            "main": (self.main, np.uint8), "tail2": (self.tail2, np.uint8),
            "tail4": (self.tail4, np.uint8), "secondary": (self.secondary, np.uint8),
            "meta": (self.meta, np.uint16), "sorder_zero2": (self.sorder_zero2, np.uint8),
            "sorder_scale2": (self.sorder_scale2, np.uint16),
            "fourbit_scale": (self.fourbit_scale, np.uint16),
            "fourbit_zero": (self.fourbit_zero, np.uint8),
            "csr_row_ptr": (self.row_ptr, np.uint32), "csr_col_ind": (self.col_ind, np.uint16),
            "csr_values": (self.values, np.uint16),
        }
        keep = []
        ctype = {np.uint8: C.c_uint8, np.uint16: C.c_uint16, np.uint32: C.c_uint32}
        for name, (arr, dt) in arrays.items():
            a = np.ascontiguousarray(arr, dtype=dt)
            keep.append(a)
            setattr(v, name, a.ctypes.data_as(C.POINTER(ctype[dt])))
        v.plan_bits_len, v.plan_perm_len = self.plan_bits.size, self.plan_perm.size
        v.main_len, v.tail2_len, v.tail4_len = self.main.size, self.tail2.size, self.tail4.size
        v.secondary_len, v.meta_len = self.secondary.size, self.meta.size
        v.sorder_len, v.fourbit_len = self.sorder_zero2.size, self.fourbit_zero.size
        v.csr_row_ptr_len, v.csr_nnz = self.row_ptr.size, self.col_ind.size
        self._keep = keep
        v._owner = self  # noqa: keep arrays alive with the view
        return v

    @classmethod
    def _from_handle(cls, h: C.c_void_p) -> "PackedLayer":
        v = LayerView()
        check(lib().qw_host_view(h, C.byref(v)))

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

        cfg = LayerConfig(rows=v.rows, cols=v.cols, n4=v.n4, pad2=v.pad2,
                          outlier_count=v.outlier_count, group2=v.group2, alpha=v.alpha,
                          outlier_ratio=v.outlier_ratio, n=v.n, n2=v.n2, group1=v.group1,
                          tile=v.tile)
        out = cls(cfg=cfg,
                  plan_bits=arr(v.plan_bits, v.plan_bits_len, np.uint8),
                  plan_perm=arr(v.plan_perm, v.plan_perm_len, np.uint32),
                  main=arr(v.main, v.main_len, np.uint8),
                  tail2=arr(v.tail2, v.tail2_len, np.uint8),
                  tail4=arr(v.tail4, v.tail4_len, np.uint8),
                  secondary=arr(v.secondary, v.secondary_len, np.uint8),
                  meta=arr(v.meta, v.meta_len, np.uint16),
                  sorder_zero2=arr(v.sorder_zero2, v.sorder_len, np.uint8),
                  sorder_scale2=arr(v.sorder_scale2, v.sorder_len, np.uint16),
                  fourbit_scale=arr(v.fourbit_scale, v.fourbit_len, np.uint16),
                  fourbit_zero=arr(v.fourbit_zero, v.fourbit_len, np.uint8),
                  row_ptr=arr(v.csr_row_ptr, v.csr_row_ptr_len, np.uint32),
                  col_ind=arr(v.csr_col_ind, v.csr_nnz, np.uint16),
                  values=arr(v.csr_values, v.csr_nnz, np.uint16))
        lib().qw_host_free(h)
        return out

    @classmethod
    def from_view(cls, v: LayerView) -> "PackedLayer":
        """Copy + validate_layer an external view (e.g. the reference's)."""
        h = C.c_void_p()
        check(lib().qw_host_from_view(C.byref(v), C.byref(h)))
        return cls._from_handle(h)

    def _handle(self) -> C.c_void_p:
        h = C.c_void_p()
        check(lib().qw_host_from_view(C.byref(self.view()), C.byref(h)))
        return h

    # ------------------------------------------------------------ accounting
    @property
    def nnz(self) -> int:
        return int(self.col_ind.size)

    def info(self) -> dict:
        inf = LayerInfo()
        check(lib().qw_layer_view_info(C.byref(self.view()), C.byref(inf)))
        return inf.as_dict()

    def streams_equal(self, other: "PackedLayer") -> bool:
        names = ("plan_bits", "plan_perm", "main", "tail2", "tail4", "secondary", "meta",
                 "sorder_zero2", "sorder_scale2", "fourbit_scale", "fourbit_zero", "row_ptr",
                 "col_ind", "values")
        same = all(np.array_equal(getattr(self, n), getattr(other, n)) for n in names)
        a, b = self.cfg, other.cfg
        return same and (a.rows, a.cols, a.n4, a.pad2, a.outlier_count, a.group2) == \
            (b.rows, b.cols, b.n4, b.pad2, b.outlier_count, b.group2)


# ---------------------------------------------------------------- producer
def synth_gaussian(rows: int, cols: int, seed: int) -> np.ndarray:
    """synth_gaussian (synth.cpp:11-21): rows x cols N(0,1) fp32."""
    out = np.empty((rows, cols), dtype=np.float32)
    check(lib().qw_synth_gaussian(rows, cols, seed, out.ctypes.data))
    return out


def plant_outliers(w: np.ndarray, ratio: float, scale: float, seed: int) -> None:
    """plant_outliers (synth.cpp:23-37), in place."""
    if w.dtype != np.float32 or not w.flags.c_contiguous:
        raise QWeightError(1, "plant_outliers: need a contiguous float32 array")
    check(lib().qw_plant_outliers(w.ctypes.data, w.size, ratio, scale, seed))


def synth_calibration(cols: int, seed: int) -> np.ndarray:
    out = np.empty(cols, dtype=np.float32)
    check(lib().qw_synth_calibration(cols, seed, out.ctypes.data))
    return out


def synth_activation(cols: int, seed: int) -> np.ndarray:
    out = np.empty(cols, dtype=np.float32)
    check(lib().qw_synth_activation(cols, seed, out.ctypes.data))
    return out


def quantize_layer(w: np.ndarray, h: np.ndarray, alpha: float = 0.25, group2: int = 16,
                   outlier_ratio: float = 0.002, threads: int = 0) -> PackedLayer:
    """quantize_layer (quantizer.hpp:21-22; QuantizeParams defaults 13-17)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    h = np.ascontiguousarray(h, dtype=np.float32)
    if w.ndim != 2 or h.shape != (w.shape[1],):
        raise QWeightError(1, "quantize_layer: w must be rows x cols and h length cols")
    hd = C.c_void_p()
    check(lib().qw_host_quantize(w.ctypes.data, w.shape[0], w.shape[1], h.ctypes.data,
                                 float(alpha), int(group2), float(outlier_ratio), int(threads),
                                 C.byref(hd)))
    return PackedLayer._from_handle(hd)


def quantize_layer_gpu(w: np.ndarray, h: np.ndarray, alpha: float = 0.25, group2: int = 16,
                       outlier_ratio: float = 0.002, device: int = 0) -> PackedLayer:
    """quantize_layer with its data-parallel passes on the GPU (qw_device_quantize):
    the same PackedLayer as quantize_layer, bit for bit."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    h = np.ascontiguousarray(h, dtype=np.float32)
    out = C.c_void_p()
    check(lib().qw_device_quantize(w.ctypes.data, w.shape[0], w.shape[1], h.ctypes.data, alpha, group2,
                                   outlier_ratio, device, C.byref(out)))
    return PackedLayer._from_handle(out)


def synth_layer(rows: int, cols: int, seed: int = 7, alpha: float = 0.25, group2: int = 16,
                outlier_ratio: float = 0.002, threads: int = 0) -> PackedLayer:
    """The benchmark recipe: W = synth_gaussian(seed), H = synth_calibration(seed)."""
    return quantize_layer(synth_gaussian(rows, cols, seed), synth_calibration(cols, seed),
                          alpha, group2, outlier_ratio, threads)


def validate_layer(layer: PackedLayer) -> None:
    check(lib().qw_validate_layer(C.byref(layer.view())))


def payload_bytes(layer: PackedLayer) -> int:
    return int(lib().qw_payload_bytes(C.byref(layer.view())))


def write_packed_layer(layer: PackedLayer, path: str) -> None:
    h = layer._handle()
    try:
        check(lib().qw_host_write(h, str(path).encode()))
    finally:
        lib().qw_host_free(h)


def read_packed_layer(path: str) -> PackedLayer:
    h = C.c_void_p()
    check(lib().qw_host_read(str(path).encode(), C.byref(h)))
    return PackedLayer._from_handle(h)


def shard_rows(layer: PackedLayer, r0: int, r1: int) -> PackedLayer:
    """Column-parallel TP shard: output rows [r0, r1)."""
    h = layer._handle()
    out = C.c_void_p()
    try:
        check(lib().qw_host_shard_rows(h, r0, r1, C.byref(out)))
    finally:
        lib().qw_host_free(h)
    return PackedLayer._from_handle(out)


def shard_tiles(layer: PackedLayer, t0: int, t1: int):
    """Row-parallel TP shard over tiles [t0, t1).  Returns (shard, slots) where
    slots are the parent's permuted slots feeding the shard's channels, in
    the shard's channel order."""
    h = layer._handle()
    out = C.c_void_p()
    offs = (C.c_uint32 * 4)()
    try:
        check(lib().qw_host_shard_tiles(h, t0, t1, C.byref(out), offs))
    finally:
        lib().qw_host_free(h)
    shard = PackedLayer._from_handle(out)
    slots = np.concatenate([np.arange(offs[0], offs[1]), np.arange(offs[2], offs[3])])
    return shard, slots.astype(np.int64)


def permute(layer: PackedLayer, x: np.ndarray) -> np.ndarray:
    """apply_permutation (plan.cpp:107-116) in numpy: pads read 0."""
    x = np.asarray(x, dtype=np.float32)
    perm = layer.plan_perm.astype(np.int64)
    out = np.zeros(perm.size, dtype=np.float32)
    real = perm != PAD
    out[real] = x[perm[real]]
    return out
